"""Small driver for ncu: runs the config-2 pipeline on `--batch` graphs
`--iters` times after one warm-up (profile with -s to skip the warm-up)."""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--d-dtype", default="uint8", choices=["uint8", "int32"])
ap.add_argument("--lib", default=None, help="another build of the library (A/B)")
args = ap.parse_args()
if args.lib:
    from paper_2308_07403_b200 import _lib as L  # noqa: E402

    L._lib = L.load_library(args.lib)

bits, gammas, _ = wl.cfg2_batch(args.batch)
dev = torch.device("cuda", 0)
buf = B.BatchBuffers.allocate(1024, args.batch, dev, d_dtype=args.d_dtype)
buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
buf.gammas.copy_(torch.from_numpy(gammas))
B.run_chunk(buf, args.batch)
torch.cuda.synchronize()
for _ in range(args.iters):
    B.run_chunk(buf, args.batch)
torch.cuda.synchronize()
print("ok")
