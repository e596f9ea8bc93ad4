"""Host checks of the block-sparse Gauss-Jordan plan (csrc/gj_invert.cu
gj_plan_kernel, restated in batch.gj_plan_tiles): the symbolic block
pattern is a superset of the numerical one at every step, and an inversion
that skips the planned-out tiles equals the dense one (CPU, numpy)."""

import numpy as np
import pytest

from paper_2308_07403_b200 import batch as B
from paper_2308_07403_b200 import workloads as wl


def _block_gj(m, b, skip):
    """Blocked Gauss-Jordan (the K2 step order: D = A_pp^-1, A_pJ = D A_pJ,
    A_IJ -= A_Ip A_pJ, A_Ip = -A_Ip D) with block size b. With skip, tiles the
    symbolic plan leaves out are not computed. Returns (inverse, tiles run,
    symbolic pattern never missed a numerically non-zero panel block)."""
    a = m.copy()
    nt = a.shape[0] // b
    blk = lambda I, J: a[I * b:(I + 1) * b, J * b:(J + 1) * b]  # noqa: E731
    S = np.array([[np.any(blk(I, J) != 0) for J in range(nt)] for I in range(nt)])
    S[np.arange(nt), np.arange(nt)] = True
    ok, tiles = True, [0, 0, 0]
    for k in range(nt):
        d = np.linalg.inv(blk(k, k))
        tiles[0] += 1
        rowp = [J for J in range(nt) if J != k and S[k, J]]
        colp = [I for I in range(nt) if I != k and S[I, k]]
        for J in range(nt):
            if J != k and np.any(blk(k, J) != 0) and not S[k, J]:
                ok = False
        for I in range(nt):
            if I != k and np.any(blk(I, k) != 0) and not S[I, k]:
                ok = False
        rows = colp if skip else [I for I in range(nt) if I != k]
        cols = rowp if skip else [J for J in range(nt) if J != k]
        for J in cols:
            a[k * b:(k + 1) * b, J * b:(J + 1) * b] = d @ blk(k, J)
            tiles[1] += 1
        for I in rows:
            aip = blk(I, k).copy()
            for J in cols:
                a[I * b:(I + 1) * b, J * b:(J + 1) * b] -= aip @ blk(k, J)
                tiles[2] += 1
            a[I * b:(I + 1) * b, k * b:(k + 1) * b] = -(aip @ d)
            tiles[2] += 1
        a[k * b:(k + 1) * b, k * b:(k + 1) * b] = d
        for I in colp:
            for J in rowp:
                S[I, J] = True
    return a, tiles, ok


def _patterns(n, rng):
    i, j = np.indices((n, n))
    out = {
        "band": (np.abs(i - j) <= 3) & (rng.random((n, n)) < 0.8),
        "two_components": ((i < n // 2) == (j < n // 2)) & (rng.random((n, n)) < 0.1),
        "dag": (i > j) & (rng.random((n, n)) < 0.05),
        "lattice": wl.lattice_present(int(np.sqrt(n)), 0.8, 3),
        "er": rng.random((n, n)) < 0.05,
        "empty": np.zeros((n, n), bool),
    }
    for p in out.values():
        np.fill_diagonal(p, False)
    return out


@pytest.mark.parametrize("name", ["band", "two_components", "dag", "lattice", "er", "empty"])
def test_skipping_planned_out_tiles_is_exact(name):
    n, b = 64, 8
    rng = np.random.default_rng(7)
    p = _patterns(n, rng)[name]
    m = np.eye(n) - 0.05 * p
    dense, td, ok_d = _block_gj(m, b, skip=False)
    sparse, ts, ok_s = _block_gj(m, b, skip=True)
    assert ok_d and ok_s, "symbolic pattern missed a non-zero block"
    np.testing.assert_array_equal(sparse, dense)
    nt = n // b
    assert td == [nt, nt * (nt - 1), nt * nt * (nt - 1)]
    # the host restatement of gj_plan_kernel counts the same tiles
    pat = np.array([[p[I * b:(I + 1) * b, J * b:(J + 1) * b].any() for J in range(nt)] for I in range(nt)])
    assert B.gj_plan_tiles(pat[None]).tolist() == [ts]


def test_dense_pattern_is_nt_cubed():
    nt = 8
    t = B.gj_plan_tiles(np.ones((3, nt, nt), bool))
    assert (t == [nt, nt * (nt - 1), nt * nt * (nt - 1)]).all()
    assert t.sum(axis=1).tolist() == [nt**3] * 3


def test_block_pattern_from_bits_matches_dense_pattern():
    rng = np.random.default_rng(1)
    for n in (300, 1024):
        i, j = np.indices((n, n))
        pres = [rng.random((n, n)) < 0.002, (np.abs(i - j) <= 40) & (rng.random((n, n)) < 0.3)]
        for q in pres:
            np.fill_diagonal(q, False)
        bits = np.stack([wl.pack_bits(q) for q in pres])
        got = B.block_pattern(bits, n)
        nt = (n + 127) // 128
        qp = [np.pad(q, ((0, nt * 128 - n), (0, nt * 128 - n))) for q in pres]
        want = np.stack([q.reshape(nt, 128, nt, 128).any(axis=(1, 3)) for q in qp])
        np.testing.assert_array_equal(got, want)


def test_cfg2_lattice_half_runs_about_half_the_tiles():
    bits, _, seeds = wl.cfg2_batch(256)
    t = B.gj_plan_tiles(B.block_pattern(bits, 1024)).sum(axis=1)
    kinds = np.array([k for k, _ in seeds])
    assert (t[kinds == "er"] == 512).all()  # ER p = 0.02: every block holds edges
    assert (t[kinds == "lattice"] < 300).all()  # bandwidth 32 << 128: ~52% of the tiles
    assert B.launches_per_call(1024, 256) == 2 + 3 + 2 * 3 * 8
