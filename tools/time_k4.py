"""K4 (power iteration, critical_gain's kernel) HBM throughput on config 3's
graph (N=8192, ER p=0.5) and config 5's size class (N=16384, p=0.01):
bytes = iterations x 8 n^2 (the weight matrix read once per iteration)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _device as _d  # noqa: E402
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

# usage: python tools/time_k4.py [lib.so ...]  (A/B of library variants)
libs = sys.argv[1:] or [None]
cases = [(8192, 0.5), (16384, 0.01)]
graphs = {c: wl.er_graph(c[0], c[1], 0) for c in cases}
out = []
for path, (n, p) in [(lp, c) for lp in libs for c in cases]:
    if path:
        L._lib = L.load_library(path)
    g = graphs[(n, p)]
    w = _d.graph_weights(g)
    _d.power_iteration(w, True, 1e-6, 10 * n + 100)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    reps = 5
    for _ in range(reps):
        rho, conv, it = _d.power_iteration(w, True, 1e-6, 10 * n + 100)
    ev[1].record()
    torch.cuda.synchronize()
    t = ev[0].elapsed_time(ev[1]) / reps
    out.append({"lib": path, "n": n, "p": p, "rho": rho, "iterations": it, "ms": t, "GBps": it * 8 * n * n / t / 1e6})
    print(json.dumps(out[-1]), flush=True)
