"""K2 time of batched dense-wide inversions at n = 512 and n = 1024: Erdos-Renyi
graphs (p = 0.02: a sparse first step) and denser graphs (p = 0.3: every step
dense), to size a two-level scheme (n = 1024 as two 512-wide steps whose band
inverses are n = 512 dense-wide inversions).

usage: python tools/k2_sizes.py [--out gpurun_out/k2_sizes.json]
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


def time_k2(n, p, batch, gamma, reps=7):
    dev = torch.device("cuda", 0)
    bits = np.stack([wl.pack_bits(wl.er_present(n, p, 100 + s)) for s in range(batch)])
    gam = np.full(batch, gamma)
    buf = B.BatchBuffers.allocate(n, batch, dev)
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gam))
    sh = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        B.run_chunk(buf, batch, sh)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ts, tstep = [], []
    for _ in range(reps):
        buf.stage_build(batch, sh)
        ev[0].record()
        buf.stage_invert(batch, sh)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
        ev[2].record()
        B.run_chunk(buf, batch, sh)
        ev[3].record()
        torch.cuda.synchronize()
        tstep.append(ev[2].elapsed_time(ev[3]))
    dense, sparse = B.sparse_first_step(bits, n)
    fl = B.executed_flops(bits, n)
    k2 = float(np.median(ts))
    return {"n": n, "p": p, "batch": batch, "gamma": gamma, "k2_ms": k2, "step_ms": float(np.median(tstep)),
            "dense_wide": int(dense.sum()), "sparse_first": int(sparse.sum()), "executed_gflop": fl / 1e9,
            "tflops": fl / (k2 * 1e-3) / 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    L.load_library()
    out = []
    for n, p, batch, gamma in ((512, 0.02, 128, 1e-2), (512, 0.3, 128, 1e-3), (512, 0.02, 256, 1e-2),
                               (512, 0.3, 256, 1e-3), (1024, 0.02, 128, 1e-2), (1024, 0.3, 128, 1e-3)):
        r = time_k2(n, p, batch, gamma)
        print(json.dumps(r), flush=True)
        out.append(r)
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
