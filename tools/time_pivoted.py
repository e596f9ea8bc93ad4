"""Timing of the partial-pivoting inversion (rdb_invert_pivoted) on random
matrices that need pivoting: blocked path (n >= 256) vs the size's FP64 flop.

usage: python tools/time_pivoted.py [--sizes 512,1024,2048,4096] [--out gpurun_out/pivoted.json]
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="512,1024,2048,4096")
    ap.add_argument("--out", default=None)
    ap.add_argument("--grids", default="", help="comma-separated RDB_PIV_GRID values to compare")
    a = ap.parse_args()
    import os
    L.load_library()
    dev = torch.device("cuda", 0)
    out = []
    cases = [(int(n), g) for n in a.sizes.split(",") for g in ([""] + [x for x in a.grids.split(",") if x])]
    for n, grid in cases:
        os.environ.pop("RDB_PIV_GRID", None)
        if grid:
            os.environ["RDB_PIV_GRID"] = grid
        g = torch.Generator(device=dev).manual_seed(n)
        m0 = torch.rand((n, n), generator=g, device=dev, dtype=torch.float64) * 2 - 1
        m = m0.clone()
        work = torch.empty(L.lib().rdb_invert_pivoted_workspace_bytes(n), dtype=torch.uint8, device=dev)
        info = L.pivot_info_tensor(1, dev)
        ts = []
        for _ in range(3):
            m.copy_(m0)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e[0].record()
            L.check(L.lib().rdb_invert_pivoted(m.data_ptr(), n, n, work.data_ptr(), info.data_ptr(),
                                               L.stream_handle()), "rdb_invert_pivoted")
            e[1].record()
            torch.cuda.synchronize()
            ts.append(e[0].elapsed_time(e[1]))
        res = (m @ m0 - torch.eye(n, device=dev, dtype=torch.float64)).abs().max().item()
        rec = {"n": n, "grid": grid or "default", "ms": min(ts), "tflops": 2.0 * n**3 / (min(ts) * 1e-3) / 1e12, "residual": res}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
