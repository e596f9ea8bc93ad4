"""K2 batched time split by graph family: 256 ER, 256 lattices, and the mixed
cfg2 batch (with the block-sparse plan and with the dense schedule).

usage: python tools/k2_split.py  (one JSON line per case)
"""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402


def time_case(name, bits, gammas, reps=5):
    dev = torch.device("cuda", 0)
    n = 1024
    count = bits.shape[0]
    buf = B.BatchBuffers.allocate(n, count, dev)
    buf.bits.copy_(torch.from_numpy(np.ascontiguousarray(bits).view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gammas))
    sh = torch.cuda.current_stream().cuda_stream
    B.run_chunk(buf, count, sh)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(reps):
        buf.stage_build(count, sh)
        ev[0].record()
        buf.stage_invert(count, sh)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    t = float(np.median(ts))
    fl = B.executed_flops(bits, n)
    print(json.dumps({"case": name, "skip": os.environ.get("RDB_GJ_SKIP", "1"), "graphs": count, "k2_ms": t,
                      "executed_flop": fl, "executed_tflops": fl / t / 1e9,
                      "dense_equiv_tflops": 2 * 1024**3 * count / t / 1e9}), flush=True)
    del buf
    torch.cuda.empty_cache()


def main():
    if len(sys.argv) > 1:  # a variant library (make BUILD=... LIB=tools/_var/x.so EXTRA=-D...)
        from paper_2308_07403_b200 import _lib as L
        L._lib = L.load_library(sys.argv[1])
    bits, gammas, _ = wl.cfg2_batch(256)
    er = np.concatenate([bits[:128], bits[:128]])
    lat = np.concatenate([bits[128:], bits[128:]])
    time_case("mixed", bits, gammas)
    time_case("er256", er, np.full(256, wl.cfg2_gamma("er")))
    time_case("lattice256", lat, np.full(256, wl.cfg2_gamma("lattice")))
    time_case("er128", bits[:128], gammas[:128])
    time_case("lattice128", bits[128:], gammas[128:])


if __name__ == "__main__":
    main()
