"""A/B timing of K6 (config 4 next-hop table, all 4096 targets) for library variants."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402

libs = sys.argv[1:]
L._lib = L.load_library(libs[0])
import paper_2308_07403_b200 as rb  # noqa: E402
from paper_2308_07403_b200 import _device as _d  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

c = wl.CFG4
g = wl.weighted_er_graph(c["n"], c["p"], c["w_lo"], c["w_hi"], 42)
w = _d.graph_weights(g)
r = rb.r_distance_device(rb.resolvent(g, c["gamma"], with_residual=False))
tg = torch.arange(c["n"], dtype=torch.int32, device="cuda")
nnz = _d.count_edges(w)
ref = None
for path in libs:
    L._lib = L.load_library(path)
    out = _d.next_hop(w, r, tg, nnz)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(5):
        out = _d.next_hop(w, r, tg, nnz)
    ev[1].record()
    torch.cuda.synchronize()
    same = True if ref is None else bool(torch.equal(out, ref))
    ref = out if ref is None else ref
    print(path, round(ev[0].elapsed_time(ev[1]) / 5, 3), "ms", "same" if same else "DIFFERENT", flush=True)
