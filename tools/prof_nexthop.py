"""ncu driver for K6: the config-4 next-hop table (all 4096 targets), after one warm-up."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2308_07403_b200 as rb  # noqa: E402
from paper_2308_07403_b200 import _device as _d  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

c = wl.CFG4
g = wl.weighted_er_graph(c["n"], c["p"], c["w_lo"], c["w_hi"], 42)
w = _d.graph_weights(g)
r = rb.r_distance_device(rb.resolvent(g, c["gamma"], with_residual=False))
tg = torch.arange(c["n"], dtype=torch.int32, device="cuda")
nnz = _d.count_edges(w)
for _ in range(2):
    out = _d.next_hop(w, r, tg, nnz)
torch.cuda.synchronize()
print("ok", int((out >= 0).sum()))
