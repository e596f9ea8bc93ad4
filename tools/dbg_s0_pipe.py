"""Where the pipeline's Y (M from bits) differs from the generic entry point's."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L, batch as B, workloads as wl
if len(sys.argv) > 1 and sys.argv[1] != "-":
    L._lib = L.load_library(sys.argv[1])
import os
for n, p, count in ((512, 0.03, 12), (1024, 0.02, 12), (1536, 0.012, 12)):
  print("n", n)
  for mode in ("default", "dense"):
    os.environ.pop("RDB_GJ_DW_S0", None)
    if mode == "dense":
        os.environ["RDB_GJ_DW_S0"] = "0"
    rng = np.random.default_rng(n)
    presents = []
    for k in range(count):
        q = rng.random((n, n)) < p
        if k == 5:
            q[n - 7, :200] = True
        np.fill_diagonal(q, False)
        presents.append(q)
    bits = np.stack([wl.pack_bits(q) for q in presents])
    gam = np.full(count, 1e-2)
    dev = torch.device("cuda")
    sh = torch.cuda.current_stream().cuda_stream
    fill = float(sys.argv[2]) if len(sys.argv) > 2 else None
    buf = B.BatchBuffers.allocate(n, count, dev)
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gam))
    buf.stage_build(count, sh)
    buf.stage_invert(count, sh)
    torch.cuda.synchronize()
    y = buf.m.clone()
    if fill is not None:
        buf.m.fill_(fill)
    if len(sys.argv) > 3:
        buf.work.fill_(int(sys.argv[3]))
    B.run_chunk(buf, count, sh)
    torch.cuda.synchronize()
    yp = buf.m
    for b in range(count):
        d = (y[b] != yp[b])
        if d.any():
            idx = d.nonzero()
            print("graph", b, "differing entries", int(d.sum()), "rows", int(idx[:, 0].min()), int(idx[:, 0].max()), "cols",
                  int(idx[:, 1].min()), int(idx[:, 1].max()), "max rel", float(((y[b] - yp[b]).abs() / y[b].abs().clamp_min(1e-300)).max()))
    del buf
  import paper_2308_07403_b200 as rb
  got = rb.rounded_r_distance_batch(bits[5:6], gam[5:6], n)[0]
  print("single", got.shape)
print("done")
