"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package ``rdist`` from
/root/reference/pkg/src, feeds it seeded inputs built with this repo's
generators (whose ER pattern is the reference's own gen_random_dense
recipe — checked below), and writes compressed .npz fixtures next to this
file. Tests compare the oracle (CPU) and the CUDA path (GPU) against them;
nothing at test / bench time reads /root/reference.

Environment recorded in meta.json: numpy/scipy versions and BLAS threads.
"""

from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import rdist  # noqa: E402  (the reference)
import scipy  # noqa: E402

from paper_2308_07403_b200 import workloads as wl  # noqa: E402


def whash(w: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(w, dtype=np.float64).tobytes()).hexdigest()[:16]


def d_u8(d: np.ndarray) -> np.ndarray:
    """fp64 D (small non-negative ints, +inf) -> uint8 with 255 for inf."""
    out = np.full(d.shape, 255, dtype=np.uint8)
    fin = np.isfinite(d)
    assert (d[fin] < 255).all() and (d[fin] == np.round(d[fin])).all()
    out[fin] = d[fin].astype(np.uint8)
    return out


def min_gap(r: np.ndarray) -> float:
    off = ~np.eye(r.shape[0], dtype=bool) & np.isfinite(r)
    g = np.abs(r[off] - np.round(r[off]))
    g = g[g > 0]
    return float(g.min()) if g.size else math.inf


def ug(w):
    return rdist.Graph(w.shape[0], w, rdist.GraphKind.UNWEIGHTED)


def main() -> None:
    out: dict[str, dict[str, np.ndarray]] = {}
    meta: dict[str, object] = {
        "numpy": np.__version__,
        "scipy": scipy.__version__,
        "reference": "/root/reference/pkg/src/rdist (rdist " + rdist.__version__ + ")",
    }
    try:
        from threadpoolctl import threadpool_info

        meta["blas"] = [{k: i.get(k) for k in ("internal_api", "version", "num_threads")} for i in threadpool_info()]
    except Exception:  # noqa: BLE001
        pass

    # --- known-answer tests from the reference's own test suite -------------
    chain2 = rdist.graph_from_edge_list(rdist.EdgeList(2, ((0, 1, 1.0),)), rdist.GraphKind.UNWEIGHTED)
    ring3 = rdist.graph_from_edge_list(
        rdist.EdgeList(3, tuple((i, (i + 1) % 3, 1.0) for i in range(3))), rdist.GraphKind.UNWEIGHTED
    )
    grid4 = rdist.gen_grid(4)
    kat = {
        "chain2_w": chain2.weights,
        "chain2_y": rdist.resolvent(chain2, 0.5).y,
        "chain2_r": rdist.r_distance(rdist.resolvent(chain2, 0.5)),
        "ring3_w": ring3.weights,
        "ring3_y_0p1": rdist.resolvent(ring3, 0.1).y,
        "grid4_w": grid4.weights,
        "grid4_d_1em3": rdist.rounded_r_distance(rdist.resolvent(grid4, 1e-3)),
        "grid4_bfs": rdist.bfs_apsp(grid4),
        "exact_power_r": rdist.r_distance(
            rdist.ResolventResult(np.array([[1.0, 0.3**2], [0.3, 1.0]]), 0.3, rdist.HealthFlags(False, None, 0.0))
        ),
        "complete7_rho": np.array(rdist.spectral_radius(np.ones((7, 7)) - np.eye(7), tol=1e-8)),
        "k11_gc": np.array(rdist.critical_gain(rdist.gen_random_dense(11, 1.0, 0))),
    }
    rng = np.random.default_rng(7)
    gen = (rng.uniform(-10, 10, (5, 5)) + 20 * np.eye(5))
    kat["generic5_m"] = gen
    kat["generic5_inv"] = rdist.lu_invert(gen)
    out["kat"] = kat

    # --- config 1: N=512 ER p=0.05 gamma=1e-3 (full size) --------------------
    c = wl.CFG1
    g_ref = rdist.gen_random_dense(c["n"], c["p"], 0)
    w1 = wl.er_graph(c["n"], c["p"], 0).weights
    assert np.array_equal(g_ref.weights, w1), "ER generator must reproduce gen_random_dense"
    res = rdist.resolvent(g_ref, c["gamma"])
    r1 = rdist.r_distance(res)
    d1 = np.ceil(r1)
    bfs1 = rdist.bfs_apsp(g_ref)
    fw1 = rdist.floyd_warshall(g_ref)
    assert np.array_equal(d1, bfs1) and np.array_equal(bfs1, fw1)
    pi = rdist.power_iteration(rdist.adjacency_indicator(g_ref))
    out["cfg1"] = {
        "seed": np.array(0),
        "w_hash": np.array(whash(w1)),
        "d": d_u8(d1),
        "r": r1,
        "residual": np.array(res.health.inversion_residual),
        "min_gap": np.array(min_gap(r1)),
        "rho": np.array(pi.value),
        "rho_iters": np.array(pi.iterations),
        "critical_gain": np.array(rdist.critical_gain(g_ref)),
    }

    # --- config 2 samples: ER + lattices at N=1024 ----------------------------
    for kind, seed in (("er", 2000), ("lattice", 1000), ("lattice", 1001), ("lattice", 1004)):
        w = wl.weights_from_present(wl.cfg2_present(kind, seed))
        gamma = wl.cfg2_gamma(kind)
        r = rdist.r_distance(rdist.resolvent(ug(w), gamma, with_residual=False))
        d = np.ceil(r)
        off = np.isfinite(r) & ~np.eye(w.shape[0], dtype=bool)
        out[f"cfg2_{kind}_{seed}"] = {
            "kind": np.array(kind),
            "seed": np.array(seed),
            "gamma": np.array(gamma),
            "w_hash": np.array(whash(w)),
            "d": d_u8(d),
            "min_gap": np.array(min_gap(r)),
            "exact_int": np.array(int((r[off] == np.round(r[off])).sum())),
        }

    # --- config 4 analogue (smaller N): weighted U[1,5], R and next hops ------
    n4 = 384
    gw = wl.weighted_er_graph(n4, 0.1, 1.0, 5.0, 42)
    g4 = rdist.Graph(n4, np.array(gw.weights), rdist.GraphKind.REAL_WEIGHTED)
    r4 = rdist.r_distance(rdist.resolvent(g4, 1e-3, with_residual=False))
    nxt = np.full((n4, n4), -1, dtype=np.int16)
    for t in range(n4):
        for j in range(n4):
            pr = rdist.greedy_descent(g4, r4, j, t, max_steps=1)
            if pr.steps_taken == 1:
                nxt[t, j] = pr.vertices[1]
    paths = []
    prng = np.random.default_rng(5)
    for _ in range(64):
        s, t = (int(x) for x in prng.integers(0, n4, 2))
        pr = rdist.greedy_descent(g4, r4, s, t)
        paths.append((s, t, pr.length, int(pr.reached), pr.steps_taken, len(pr.vertices)))
    out["cfg4_small"] = {
        "n": np.array(n4),
        "seed": np.array(42),
        "gamma": np.array(1e-3),
        "w_hash": np.array(whash(gw.weights)),
        "r": r4,
        "next": nxt,
        "paths": np.array(paths, dtype=np.float64),
    }

    out.update(sweep_fixtures())
    out.update(wire_fixtures())
    write(out)
    (HERE / "meta.json").write_text(json.dumps(meta, indent=1) + "\n")


def write(out: dict[str, dict[str, np.ndarray]]) -> None:
    for name, arrays in out.items():
        np.savez_compressed(HERE / f"{name}.npz", **arrays)
    for p in sorted(HERE.glob("*.npz")):
        print(p.name, p.stat().st_size)


SWEEPS = (("grid", 64, {}), ("tree", 63, {}), ("hanoi", 81, {}), ("dense", 80, {"p": 0.1, "seed": 3}),
          ("power_law", 100, {"seed": 1}))


def sweep_fixtures() -> dict[str, dict[str, np.ndarray]]:
    """The reference's gamma sweep (experiments.sweep_gamma, per_decade=3) on
    five small graph families, the graphs stored as bit-packed patterns (the
    repo has no copy of the reference's generators), plus the reference's
    global/local accuracy of fixed estimates (raw R and its ceiling)."""
    from rdist import experiments as ex

    out = {}
    for fam, size, kw in SWEEPS:
        g = ex.build_family(fam, size, **kw)
        assert g.kind is rdist.GraphKind.UNWEIGHTED
        present = np.isfinite(g.weights) & ~np.eye(size, dtype=bool)
        recs = ex.sweep_gamma(fam, [size], per_decade=3, **kw)
        exact = rdist.bfs_apsp(g)
        gm = rdist.suggest_gamma(rdist.gamma_bounds(g, max(int(rdist.graph_diameter(exact)), 1)))
        raw = rdist.r_distance(rdist.resolvent(g, gm))
        rounded = np.ceil(raw)
        # per gamma, how many counted items sit on a numerical knife edge of the
        # reference's own arithmetic (where a different but equally accurate
        # inverse may legitimately land on the other side):
        #  global: pairs with |R - round(R)| < 1e-9 (ceil flips);
        #  local : (goal, node) whose two best successor estimates are within
        #          1e-9 relative (argmin flips);
        #  underflow: reachable pairs with 0 <= |y| < 2**-1000 (zero vs tiny).
        reach = np.isfinite(exact) & ~np.eye(size, dtype=bool)
        adj = np.isfinite(g.weights)
        frag = []
        for r in recs:
            try:
                res = rdist.resolvent(g, r.gamma, reachable=reach, with_residual=False)
            except rdist.ResolventSingularError:
                frag.append((0, 0, 0))
                continue
            rr = rdist.r_distance(res)
            fin = reach & np.isfinite(rr)
            fg = int((np.abs(rr[fin] - np.round(rr[fin])) < 1e-9).sum())
            fl = 0
            for t in range(size):
                nodes = np.flatnonzero(np.isfinite(exact[t]) & (np.arange(size) != t) & adj.any(axis=0))
                if nodes.size == 0:
                    continue
                e = np.where(adj[:, nodes], rr[t][:, None], np.inf)
                e.sort(axis=0)
                if e.shape[0] > 1:
                    b0, b1 = e[0], e[1]
                    close = np.isfinite(b1) & (np.abs(b1 - b0) <= 1e-9 * np.maximum(np.abs(b0), 1e-300))
                    fl += int(close.sum())
            fu = int((reach & (np.abs(res.y) < 2.0**-1000)).sum())
            frag.append((fg, fl, fu))
        frag = np.array(frag, dtype=np.int64)
        out[f"sweep_{fam}_{size}"] = {
            "frag_global": frag[:, 0],
            "frag_local": frag[:, 1],
            "frag_underflow": frag[:, 2],
            "evaluated_global": np.array(int(reach.sum())),
            "evaluated_local": np.array(int((reach & adj.any(axis=0)[None, :]).sum())),
            "n": np.array(size),
            "bits": wl.pack_bits(present),
            "w_hash": np.array(whash(g.weights)),
            "gamma": np.array([r.gamma for r in recs]),
            "global_fraction": np.array([r.global_fraction for r in recs]),
            "local_fraction": np.array([r.local_fraction for r in recs]),
            "negative_entries": np.array([r.negative_entries for r in recs]),
            "underflow_zeros": np.array([r.underflow_zeros for r in recs]),
            "gamma_over_critical": np.array([r.gamma_over_critical for r in recs]),
            "precision_floor": np.array([r.precision_floor for r in recs]),
            "exact": exact,
            "acc_gamma": np.array(gm),
            "acc_raw": raw,
            "acc_global_rounded": np.array(rdist.global_accuracy(rounded, exact)),
            "acc_local_raw": np.array(rdist.local_accuracy(g, raw, exact)),
            "acc_local_rounded": np.array(rdist.local_accuracy(g, rounded, exact)),
        }
    return out


def wire_fixtures() -> dict[str, dict[str, np.ndarray]]:
    """The reference's edge-list and distance-CSV formats (graphs.py:284-329,
    cli.py:204-210) on a small weighted graph and an unweighted one with
    unreachable pairs."""
    import tempfile

    from rdist import cli
    from rdist import graphs as gr

    gw = rdist.gen_weighted_dense(12, 0.3, 1.0, 100.0, 1)
    el = gr.edge_list_from_graph(gw)
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "g.txt"
        gr.write_edge_list(el, p)
        text = p.read_text()
        back = gr.read_edge_list(p)
        assert back == el
        ring = rdist.graph_from_edge_list(rdist.EdgeList(4, ((0, 1, 1.0), (1, 2, 1.0), (2, 0, 1.0))),
                                          rdist.GraphKind.UNWEIGHTED)
        d = rdist.rounded_r_distance(rdist.resolvent(ring, 0.1))
        q = Path(td) / "d.csv"
        cli._write_distance_csv(d, str(q))
        csv = q.read_text()
    return {"wire": {
        "weights": gw.weights,
        "edge_text": np.array(text),
        "edges": np.array(el.edges, dtype=np.float64),
        "kind": np.array(gr.infer_kind(el).value),
        "ring_d": d,
        "ring_csv": np.array(csv),
    }}


if __name__ == "__main__":
    if sys.argv[1:] == ["sweep"]:
        write(sweep_fixtures())
    elif sys.argv[1:] == ["wire"]:
        write(wire_fixtures())
    else:
        main()
