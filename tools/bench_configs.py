"""Per-config measurements and parity on B200 for BASELINE.json configs 1, 3, 4, 5
(config 2 is bench.py's headline workload).

  python tools/bench_configs.py --configs 1,3,4,5 [--cfg5-parity] [--out gpurun_out/configs.json]

For each config: device time of the path with inputs resident in HBM (CUDA
events), K2 inversion FP64 TFLOP/s against the measured DMMA peak, and the
reference pipeline restated in oracle/ timed on the host (median of runs, or a
single run for the big configs). Config 5 (N = 32768): the inversion of the full
8.6 GB matrix is timed; with --cfg5-parity, D on 4096 seeded sample columns is
compared bit-exact with the LAPACK restatement (lu_factor as linalg.py:32 +
lu_solve on identity columns) and with BFS from those sources.
"""

import argparse
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import paper_2308_07403_b200 as rb  # noqa: E402
from paper_2308_07403_b200 import _device as _d  # noqa: E402
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

PEAK = json.loads((ROOT / "profiles" / "r01_fp64_peak.json").read_text())["dmma_tflops_sustained"]


def ev():
    return torch.cuda.Event(enable_timing=True)


def time_device(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def pipeline_dense(w_dev, n, gamma, want_r):
    """K1 -> K2 -> K3 on a device weight matrix; returns (R or D tensor, t_inv_ms)."""
    n_pad = L.pad_to_nb(n)
    m = _d.build_m(w_dev, n, gamma, n_pad)
    rec = _d.invert_padded_nopivot(m)
    assert not rec.flags, rec.flags
    r, dc = _d.log_ceil(m, n, gamma, want_r=want_r, want_dceil=not want_r)
    return (r if want_r else dc)


def measure_dense(name, g, gamma, want_r, cpu_runs):
    n = g.n_vertices
    w = _d.graph_weights(g)
    n_pad = L.pad_to_nb(n)
    t_all = time_device(lambda: pipeline_dense(w, n, gamma, want_r))
    m = _d.build_m(w, n, gamma, n_pad)
    work = torch.empty(L.lib().rdb_invert_workspace_bytes(n_pad, 1), dtype=torch.uint8, device="cuda")
    info = L.pivot_info_tensor(1, torch.device("cuda"))
    buf = m.clone()

    def inv():
        buf.copy_(m)
        L.check(L.lib().rdb_invert(buf.data_ptr(), n_pad, n_pad, work.data_ptr(), info.data_ptr(),
                                   L.stream_handle()), "rdb_invert")

    t_copy = time_device(lambda: buf.copy_(m))
    t_inv = time_device(inv) - t_copy
    out = pipeline_dense(w, n, gamma, want_r).cpu().numpy()
    import rdist_oracle as orc

    wh = np.asarray(g.weights)
    t0 = time.perf_counter()
    for _ in range(cpu_runs):
        ref = orc.run_rdist(wh, gamma, unweighted=not want_r)
    t_cpu = (time.perf_counter() - t0) / cpu_runs
    if want_r:
        fin = np.isfinite(ref)
        ok_fin = bool(np.array_equal(np.isfinite(out), fin))
        rel = float(np.max(np.abs(out[fin] - ref[fin]) / np.maximum(np.abs(ref[fin]), 1e-300)))
        parity = {"finite_pattern_equal": ok_fin, "max_rel_err_R": rel}
    else:
        parity = {"D_bit_exact": bool(np.array_equal(out, ref)), "mismatches": int((out != ref).sum())}
    flops = 2.0 * n_pad**3
    return {
        "config": name, "n": n, "gamma": gamma, "device_ms_pipeline": t_all, "device_ms_inversion": t_inv,
        "inversion_tflops": flops / (t_inv * 1e-3) / 1e12, "frac_of_fp64_peak": flops / (t_inv * 1e-3) / 1e12 / PEAK,
        "cpu_ms_reference_pipeline": t_cpu * 1e3, "cpu_threads": orc.blas_threads(),
        "speedup_vs_cpu": t_cpu * 1e3 / t_all, "parity": parity,
    }


def cfg4(cpu_targets=256):
    c = wl.CFG4
    g = wl.weighted_er_graph(c["n"], c["p"], c["w_lo"], c["w_hi"], 42)
    res = measure_dense("cfg4", g, c["gamma"], True, 1)
    import rdist_oracle as orc

    w = _d.graph_weights(g)
    r = rb.r_distance_device(rb.resolvent(g, c["gamma"], with_residual=False))
    n = g.n_vertices
    tg = torch.arange(n, dtype=torch.int32, device="cuda")
    nnz = _d.count_edges(w)
    t_nh = time_device(lambda: _d.next_hop(w, r, tg, nnz))
    nxt = _d.next_hop(w, r, tg, nnz).cpu().numpy()
    rh = r.cpu().numpy()
    sample = np.random.default_rng(1).choice(n, cpu_targets, replace=False)
    t0 = time.perf_counter()
    ref = orc.next_hop_table(np.asarray(g.weights), rh, sample)
    t_cpu = time.perf_counter() - t0
    res["next_hop"] = {
        "device_ms_full_table": t_nh, "pairs": int(n * nnz), "pairs_per_s": n * nnz / (t_nh * 1e-3),
        "bit_exact_sampled_targets": bool(np.array_equal(nxt[sample], ref)), "sampled_targets": cpu_targets,
        "cpu_s_sampled": t_cpu, "cpu_s_full_table_extrapolated": t_cpu * n / cpu_targets,
    }
    return res


def cfg5(parity: bool, n_cols: int = 4096):
    """Config 5 on one GPU (single.py: BASELINE's seed, wide-step in-place
    inversion); D on the reference's 4096 seeded columns against the digests
    of the reference's own LAPACK columns (tests/golden/cfg5_cols.npz), and
    with --cfg5-parity all 1.07e9 pairs against the device BFS."""
    import hashlib

    from paper_2308_07403_b200 import single as S

    c = wl.CFG5
    n, gamma = c["n"], c["gamma"]
    t0 = time.perf_counter()
    bits = wl.er_bits_parallel(n, c["p"], 0)
    t_gen = time.perf_counter() - t0
    dev = torch.device("cuda")
    bits_d = torch.from_numpy(bits.view(np.int32)).to(dev)
    S.invert_in_place(S.build_m_bits(bits_d[:8192, :256].contiguous(), 8192, gamma), gamma)  # first-call setup
    m = S.build_m_bits(bits_d, n, gamma)
    work = torch.empty(L.lib().rdb_invert_workspace_bytes(n, 1), dtype=torch.uint8, device=dev)
    info = L.pivot_info_tensor(1, dev)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    L.check(L.lib().rdb_invert(m.data_ptr(), n, n, work.data_ptr(), info.data_ptr(), L.stream_handle()), "invert")
    b.record()
    torch.cuda.synchronize()
    t_inv = a.elapsed_time(b)
    rec = L.read_pivot_info(info)[0]
    flops = 2.0 * n**3
    res = {
        "config": "cfg5", "n": n, "gamma": gamma, "host_gen_s": t_gen, "device_ms_inversion": t_inv,
        "inversion_tflops": flops / (t_inv * 1e-3) / 1e12, "frac_of_fp64_peak": flops / (t_inv * 1e-3) / 1e12 / PEAK,
        "min_pivot": rec.min_pivot, "pivot_flags": rec.flags,
    }
    f = np.load(ROOT / "tests" / "golden" / "cfg5_cols.npz")
    cols = f["cols"]
    d = S.d_columns(m, n, gamma, cols)
    du = torch.where(torch.isfinite(d), d, torch.full_like(d, 255)).to(torch.uint8).cpu().numpy()
    got = np.array([hashlib.sha256(np.ascontiguousarray(du[:, k]).tobytes()).digest()[:16] for k in range(len(cols))],
                   dtype="S16")
    res["sampled_columns"] = int(len(cols))
    res["columns_differing_from_reference"] = int((got != f["col_digest"]).sum())
    res["D_values"] = np.unique(du).tolist()
    if parity:
        d32 = S.d_int32(m, n, gamma)
        del m
        torch.cuda.empty_cache()
        from paper_2308_07403_b200 import oracles

        a, b = ev(), ev()
        a.record()
        bfs32, levels = oracles.bfs_apsp_bits(bits_d, n, torch.int32)
        b.record()
        torch.cuda.synchronize()
        res["device_ms_bfs_all_sources"] = a.elapsed_time(b)
        res["bfs_levels"] = levels
        res["D_equals_device_BFS_all_pairs"] = bool(torch.equal(d32, bfs32))
        res["pairs_checked"] = n * n
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4,5")
    ap.add_argument("--cfg5-parity", action="store_true")
    ap.add_argument("--out", default="gpurun_out/configs.json")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    rb.load_library()
    out = {"peak_tflops": PEAK, "gpu": torch.cuda.get_device_name(), "host_cpus": os.cpu_count(), "results": []}
    for c in a.configs.split(","):
        c = c.strip()
        t0 = time.perf_counter()
        if c == "1":
            r = measure_dense("cfg1", wl.er_graph(512, 0.05, 0), 1e-3, False, 5)
        elif c == "3":
            r = measure_dense("cfg3", wl.er_graph(8192, 0.5, 0), 1e-5, False, 1)
        elif c == "4":
            r = cfg4()
        elif c == "5":
            r = cfg5(a.cfg5_parity)
        else:
            continue
        r["wall_s"] = time.perf_counter() - t0
        out["results"].append(r)
        print(json.dumps(r), flush=True)
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
