"""Gamma sweep on B200 vs the reference pipeline restated
on the host: one config-2 ER graph (N=1024, p=0.02, seed 2000), a log grid of
gammas from the graph's own bounds, every point = resolvent (with residual
and the reachable mask, as _sweep_point calls it) -> R -> ceil -> global and
local accuracy. Exact distances by BFS (K8 on the device, the oracle's BFS on
the host). The CPU side runs a bounded sample of points and is extrapolated.

  python tools/bench_sweep.py [--points 64] [--cpu-points 2] [--out gpurun_out/sweep.json]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import paper_2308_07403_b200 as rb  # noqa: E402
import rdist_oracle as orc  # noqa: E402
from paper_2308_07403_b200 import sweep  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402


def cpu_point(w, exact, reach, gamma):
    y = orc.resolvent_y(w, gamma)
    neg, under = orc.health(y, reach)
    m = np.eye(w.shape[0]) - orc.build_x(w, gamma)
    orc.residual(m, y)
    raw = orc.r_distance(y, gamma)
    return orc.global_accuracy(np.ceil(raw), exact), orc.local_accuracy(w, raw, exact), neg, under


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=64)
    ap.add_argument("--cpu-points", type=int, default=2)
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    a = ap.parse_args()
    rb.load_library()
    present = wl.cfg2_present("er", 2000)
    w = wl.weights_from_present(present)
    g = rb.Graph(1024, w, rb.GraphKind.UNWEIGHTED)
    st = sweep._GraphState(g)
    finite = st.exact[torch.isfinite(st.exact)]
    bounds = rb.gamma_bounds(g, max(int(finite.max().item()), 1))
    grid = np.geomspace(max(bounds.precision_floor_for_dmax, 1e-300), min(2 * bounds.critical_gain, 0.99), a.points)
    sweep.sweep_gamma_graph(g, grid[:2])  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    recs = sweep.sweep_gamma_graph(g, grid)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    exact = orc.bfs_apsp(w)
    reach = np.isfinite(exact) & ~np.eye(1024, dtype=bool)
    pick = np.linspace(0, a.points - 1, a.cpu_points).round().astype(int)
    t0 = time.perf_counter()
    cpu = [cpu_point(w, exact, reach, grid[i]) for i in pick]
    t_cpu = (time.perf_counter() - t0) / len(pick)
    agree = [abs(recs[i].global_fraction - c[0]) < 1e-12 and abs(recs[i].local_fraction - c[1]) < 1e-12
             for i, c in zip(pick, cpu)]
    out = {
        "workload": "gamma sweep, cfg2 ER graph N=1024 p=0.02 seed 2000, resolvent with residual + reachable mask",
        "points": a.points, "gamma_range": [float(grid[0]), float(grid[-1])],
        "gpu_s_total": t_gpu, "gpu_ms_per_point": t_gpu / a.points * 1e3,
        "cpu_s_per_point": t_cpu, "cpu_points_timed": len(pick), "cpu_threads": orc.blas_threads(),
        "speedup_per_point": t_cpu / (t_gpu / a.points),
        "sampled_points_agree_with_oracle": agree,
        "records_head": [r.__dict__ for r in recs[:3]],
    }
    print(json.dumps(out), flush=True)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
