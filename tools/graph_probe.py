"""Eager launches vs one CUDA-graph replay of the config-2 pipeline
(rdb_apsp_bits_batched_d8 on 256 graphs: ~300 kernels on the caller's stream
and the library's internal sub-batch / look-ahead streams, joined back by events,
so the whole call is capturable). D must be identical.

usage: python tools/graph_probe.py [--out gpurun_out/graph_probe.json]
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    L.load_library()
    dev = torch.device("cuda", 0)
    bits, gammas, _ = wl.cfg2_batch(256)
    buf = B.BatchBuffers.allocate(1024, 256, dev, d_dtype="uint8")
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gammas))
    s = torch.cuda.Stream()
    out = {}
    with torch.cuda.stream(s):
        for _ in range(3):
            B.run_chunk(buf, 256, s.cuda_stream)
        torch.cuda.synchronize()
        ref = buf.d.clone()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(s)
        for _ in range(a.reps):
            B.run_chunk(buf, 256, s.cuda_stream)
        ev[1].record(s)
        torch.cuda.synchronize()
        out["eager_ms"] = ev[0].elapsed_time(ev[1]) / a.reps
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        B.run_chunk(buf, 256, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    buf.d.zero_()
    g.replay()
    torch.cuda.synchronize()
    out["graph_d_identical"] = bool(torch.equal(buf.d, ref))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(a.reps):
        g.replay()
    ev[1].record()
    torch.cuda.synchronize()
    out["graph_ms"] = ev[0].elapsed_time(ev[1]) / a.reps
    print(json.dumps(out), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
