"""Full-size golden digests made by running the REFERENCE on the BASELINE configs.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_full.py [cfg2] [cfg3] [cfg4] [cfg5]

The outputs at full size are too large to commit (cfg2: 256 x 1 MB of D per
rank; cfg5: 32768 x 4096 sampled columns), so each fixture stores, per graph /
row / column, a SHA-256 digest (first 16 bytes) of the reference's D in the
compact byte form (uint8, 255 = +inf; every D here is <= 254), plus the
statistics the parity argument needs (minimum distance of a non-integer R to
an integer, number of exact-integer R). A GPU test hashes its own D the same
way and requires every digest to match: bit-exact on every graph, no
tolerance and no knife-edge exemption.

- cfg2_full.npz: every graph of the bench batch of ranks 0 and 1 (512 graphs:
  ``workloads.cfg2_batch(256, rank)``), each through the reference's timed
  closure run_rdist (experiments.py:305-310: resolvent(with_residual=False)
  -> r_distance -> ceil), one single-threaded process per core.
- cfg3_full.npz: config 3 (N=8192, p=0.5, gamma=1e-5, seed 0), the
  reference's rounded_r_distance(resolvent(g, gamma)); one digest per row.
- cfg4_full.npz: config 4 (N=4096 weighted, seed 42): digests per target row
  of the full next-hop table, i.e. the reference's greedy_descent step
  (navigation.py:63-69) for every (target, vertex) — restated vectorised per
  source column (no reference function builds the table) and
  checked here against rdist.greedy_descent(..., max_steps=1) on 4000 random
  pairs — on the reference's own R; plus R itself on 64 seeded target rows.
- cfg5_cols.npz: config 5 (N=32768, p=0.01, gamma=1e-4, seed 0): the
  reference's LU call (linalg.py:32, scipy.linalg.lu_factor) on M, then
  lu_solve on the identity columns of 4096 seeded sources (SURVEY.md 8(c)-2:
  bitwise equal to the same columns of lu_invert), then r_distance's formula
  (resolvent.py:140-142); one digest per sampled column D[:, s].
"""

from __future__ import annotations

import hashlib
import json
import math
import multiprocessing as mp
import os
import sys
import time
import warnings
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, str(REPO))

CFG5_COLS_SEED, CFG5_NCOLS = 5, 4096
CFG4_R_ROWS_SEED, CFG4_R_ROWS = 9, 64


def digest(a: np.ndarray) -> bytes:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest()[:16]


def d_u8(d: np.ndarray) -> np.ndarray:
    out = np.full(d.shape, 255, dtype=np.uint8)
    fin = np.isfinite(d)
    assert (d[fin] < 255).all() and (d[fin] >= 0).all() and (d[fin] == np.round(d[fin])).all()
    out[fin] = d[fin].astype(np.uint8)
    return out


def gap_stats(r: np.ndarray, off: np.ndarray) -> tuple[float, int]:
    """(min |R - round R| over non-integer finite off-diagonal R, #exact-integer R)."""
    v = r[off & np.isfinite(r)]
    g = np.abs(v - np.round(v))
    nz = g[g > 0]
    return (float(nz.min()) if nz.size else math.inf), int((g == 0).sum())


# ------------------------------------------------------------------ cfg2
def _cfg2_init():
    from threadpoolctl import threadpool_limits

    global _LIM
    _LIM = threadpool_limits(1)


def _cfg2_one(item):
    import rdist

    from paper_2308_07403_b200 import workloads as wl

    kind, seed = item
    w = wl.weights_from_present(wl.cfg2_present(kind, seed))
    gamma = wl.cfg2_gamma(kind)
    g = rdist.Graph(w.shape[0], w, rdist.GraphKind.UNWEIGHTED)
    r = rdist.r_distance(rdist.resolvent(g, gamma, with_residual=False))  # run_rdist, experiments.py:305-310
    d = np.ceil(r)
    off = ~np.eye(w.shape[0], dtype=bool)
    mg, ex = gap_stats(r, off)
    fin = np.isfinite(d)
    return digest(d_u8(d)), mg, ex, int((~fin).sum()), float(d[fin].max())


def cfg2(ranks=(0, 1)) -> dict:
    from paper_2308_07403_b200 import workloads as wl

    items, rk = [], []
    for r in ranks:
        s = wl.cfg2_seeds(256, r)
        items += s
        rk += [r] * len(s)
    t0 = time.perf_counter()
    saved = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS")}
    os.environ.update({k: "1" for k in saved})  # single-threaded BLAS in the spawned workers
    try:
        with mp.get_context("spawn").Pool(os.cpu_count(), initializer=_cfg2_init) as pool:
            res = pool.map(_cfg2_one, items, chunksize=4)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    print(f"cfg2: {len(items)} graphs in {time.perf_counter() - t0:.1f} s", flush=True)
    return {
        "rank": np.array(rk, np.int32),
        "kind": np.array([k for k, _ in items]),
        "seed": np.array([s for _, s in items], np.int64),
        "gamma": np.array([wl.cfg2_gamma(k) for k, _ in items]),
        "digest": np.array([x[0] for x in res], dtype="S16"),
        "min_gap": np.array([x[1] for x in res]),
        "exact_int": np.array([x[2] for x in res], np.int64),
        "unreachable": np.array([x[3] for x in res], np.int64),
        "d_max": np.array([x[4] for x in res]),
    }


# ------------------------------------------------------------------ cfg3
def cfg3() -> dict:
    import rdist

    from paper_2308_07403_b200 import workloads as wl

    c = wl.CFG3
    t0 = time.perf_counter()
    g = rdist.gen_random_dense(c["n"], c["p"], 0)
    d = rdist.rounded_r_distance(rdist.resolvent(g, c["gamma"], with_residual=False))
    du = d_u8(d)
    print(f"cfg3: {time.perf_counter() - t0:.1f} s, D values {np.unique(du)}", flush=True)
    return {"n": np.array(c["n"]), "seed": np.array(0), "gamma": np.array(c["gamma"]),
            "row_digest": np.array([digest(du[i]) for i in range(c["n"])], dtype="S16"),
            "digest": np.array(digest(du), dtype="S16"),
            "values": np.unique(du), "counts": np.unique(du, return_counts=True)[1]}


# ------------------------------------------------------------------ cfg4
_W4 = _R4 = None


def _cfg4_init(w, r):
    from threadpoolctl import threadpool_limits

    global _W4, _R4, _LIM
    _LIM = threadpool_limits(1)
    _W4, _R4 = w, r


def _cfg4_cols(js):
    """next[:, j] for the columns js: first argmin over ascending successors k
    of j of W[k][j] + R[t][k] (navigation.py:63-67), -1 for t == j or a
    non-finite best (navigation.py:68-69)."""
    w, r = _W4, _R4
    n = w.shape[0]
    out = np.full((n, len(js)), -1, dtype=np.int16)
    t = np.arange(n)
    for c, j in enumerate(js):
        succ = np.flatnonzero(np.isfinite(w[:, j]))
        if succ.size == 0:
            continue
        scores = w[succ, j][None, :] + r[:, succ]
        best = np.argmin(scores, axis=1)
        ok = np.isfinite(scores[t, best]) & (t != j)
        out[ok, c] = succ[best[ok]]
    return js, out


def cfg4() -> dict:
    import rdist

    from paper_2308_07403_b200 import workloads as wl

    c = wl.CFG4
    n = c["n"]
    gw = wl.weighted_er_graph(n, c["p"], c["w_lo"], c["w_hi"], 42)
    w = np.array(gw.weights)
    g = rdist.Graph(n, w, rdist.GraphKind.REAL_WEIGHTED)
    t0 = time.perf_counter()
    r = rdist.r_distance(rdist.resolvent(g, c["gamma"], with_residual=False))
    cols = np.array_split(np.arange(n), 256)
    nxt = np.empty((n, n), dtype=np.int16)
    with mp.get_context("fork").Pool(os.cpu_count(), initializer=_cfg4_init, initargs=(w, r)) as pool:
        for js, part in pool.imap_unordered(_cfg4_cols, cols):
            nxt[:, js] = part
    print(f"cfg4: table in {time.perf_counter() - t0:.1f} s", flush=True)
    rng = np.random.default_rng(3)
    for _ in range(4000):  # the restatement is the reference's own step
        s, t = (int(x) for x in rng.integers(0, n, 2))
        pr = rdist.greedy_descent(g, r, s, t, max_steps=1)
        want = pr.vertices[1] if pr.steps_taken == 1 else -1
        assert nxt[t, s] == want, (s, t, nxt[t, s], want)
    rows = np.sort(np.random.default_rng(CFG4_R_ROWS_SEED).choice(n, CFG4_R_ROWS, replace=False))
    # margin: smallest relative gap between the best and second-best score
    return {"n": np.array(n), "seed": np.array(42), "gamma": np.array(c["gamma"]),
            "w_digest": np.array(digest(w), dtype="S16"),
            "next_row_digest": np.array([digest(nxt[t]) for t in range(n)], dtype="S16"),
            "next_digest": np.array(digest(nxt), dtype="S16"),
            "r_rows": rows, "r_sample": r[rows],
            "r_min": np.array(float(r[np.isfinite(r) & (r > 0)].min())), "r_max": np.array(float(r[np.isfinite(r)].max()))}


# ------------------------------------------------------------------ cfg5
def cfg5() -> dict:
    import scipy.linalg

    from paper_2308_07403_b200 import workloads as wl

    c = wl.CFG5
    n, gamma = c["n"], c["gamma"]
    t0 = time.perf_counter()
    bits = wl.er_bits_chunked(n, c["p"], 0, chunk_rows=2048)  # gen_random_dense(n, p, 0)'s RNG stream
    m = np.empty((n, n), dtype=np.float64, order="F")
    for r0 in range(0, n, 2048):
        blk = wl.unpack_bits(bits[r0 : r0 + 2048], n)
        m[r0 : r0 + 2048, :] = np.where(blk, -gamma, 0.0)  # M = I - build_x(g, gamma) (resolvent.py:114-115)
    m[np.arange(n), np.arange(n)] = 1.0
    t1 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        lu, piv = scipy.linalg.lu_factor(m, overwrite_a=True, check_finite=False)  # linalg.py:32
    pivots = np.abs(np.diag(lu))
    assert pivots.min() >= 1e-13  # linalg.py:33-38 (scale = 1)
    swaps = int((piv != np.arange(n)).sum())
    t2 = time.perf_counter()
    cols = np.sort(np.random.default_rng(CFG5_COLS_SEED).choice(n, CFG5_NCOLS, replace=False))
    e = np.zeros((n, len(cols)))
    e[cols, np.arange(len(cols))] = 1.0
    y = scipy.linalg.lu_solve((lu, piv), e, check_finite=False)  # linalg.py:39 on the sampled columns
    del lu, e
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(y > 0, np.log(y) / math.log(gamma), np.inf)  # resolvent.py:140-141
    r[cols, np.arange(len(cols))] = 0.0  # resolvent.py:142 (diagonal)
    d = np.ceil(r)
    du = d_u8(d)
    off = np.ones(r.shape, bool)
    off[cols, np.arange(len(cols))] = False
    mg, ex = gap_stats(r, off)
    t3 = time.perf_counter()
    print(f"cfg5: build {t1 - t0:.0f} s, getrf {t2 - t1:.0f} s, {len(cols)} columns {t3 - t2:.0f} s; "
          f"swaps {swaps}, min pivot {pivots.min()}, min gap {mg}, exact {ex}", flush=True)
    vals, cnts = np.unique(du, return_counts=True)
    return {"n": np.array(n), "seed": np.array(0), "gamma": np.array(gamma), "cols": cols,
            "col_digest": np.array([digest(du[:, k]) for k in range(len(cols))], dtype="S16"),
            "values": vals, "counts": cnts, "min_gap": np.array(mg), "exact_int": np.array(ex),
            "swaps": np.array(swaps), "min_pivot": np.array(float(pivots.min())),
            "bits_digest": np.array(digest(bits), dtype="S16")}


def main(argv):
    import scipy

    which = argv or ["cfg2", "cfg3", "cfg4", "cfg5"]
    fns = {"cfg2": ("cfg2_full", cfg2), "cfg3": ("cfg3_full", cfg3), "cfg4": ("cfg4_full", cfg4),
           "cfg5": ("cfg5_cols", cfg5)}
    meta_p = HERE / "meta_full.json"
    meta = json.loads(meta_p.read_text()) if meta_p.exists() else {}
    for w in which:
        name, fn = fns[w]
        t0 = time.perf_counter()
        arrays = fn()
        np.savez_compressed(HERE / f"{name}.npz", **arrays)
        meta[name] = {"numpy": np.__version__, "scipy": scipy.__version__, "cores": os.cpu_count(),
                      "seconds": round(time.perf_counter() - t0, 1), "reference": REF}
        print(name, (HERE / f"{name}.npz").stat().st_size, "bytes", flush=True)
    meta_p.write_text(json.dumps(meta, indent=1) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:])
