"""Generic lu_invert through the partial-pivoting kernel (linalg.py:18-39 with
LAPACK getrf's partial pivoting): the blocked path (n >= 256: cooperative panel
factorisation, row swaps, DMMA updates) against LAPACK — inverse, the
singularity decision, the pivot magnitudes — on matrices that need pivoting,
sizes on and off the 128 grid; and the unblocked path it replaces, bitwise
where both see the same pivots."""

import numpy as np
import pytest
import scipy.linalg
import torch

import paper_2308_07403_b200 as rb
import rdist_oracle as orc
from paper_2308_07403_b200 import _device as _d
from paper_2308_07403_b200 import _lib as L

pytestmark = pytest.mark.gpu


def lapack_pivots(m):
    lu, piv = scipy.linalg.lu_factor(m, check_finite=False)
    return np.abs(np.diag(lu)), piv


@pytest.mark.parametrize("n", [256, 300, 384, 640, 1000, 1024])
def test_blocked_pivoted_matches_lapack(cuda, n):
    rng = np.random.default_rng(n)
    m = rng.uniform(-1.0, 1.0, (n, n))  # no dominance: pivoting is required
    got = rb.lu_invert(m)
    ref = orc.lu_invert(m)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-9, err
    assert np.abs(got @ m - np.eye(n)).max() < 1e-8
    # same pivot magnitudes as LAPACK (same pivot rows; rounding differs)
    y = torch.from_numpy(m).to(cuda)
    rec = _d.invert_pivoted(y)
    piv_abs, _ = lapack_pivots(m)
    assert rec.min_pivot == pytest.approx(piv_abs.min(), rel=1e-9)
    assert rec.flags & L.RDB_PIV_NONPOS  # a random matrix has negative pivots


def test_blocked_pivoted_singular_raises(cuda):
    rng = np.random.default_rng(3)
    n = 512
    m = rng.uniform(-1.0, 1.0, (n, n))
    m[:, 300] = m[:, 7] * 2.0 - m[:, 100]  # exactly dependent column
    with pytest.raises(orc.OracleSingular):
        orc.lu_invert(m)
    with pytest.raises(rb.SingularMatrixError):
        rb.lu_invert(m)


def test_blocked_pivoted_on_m_matrix_past_critical_gain(cuda):
    # the resolvent past the critical gain: the certificate fails and the
    # pivoted path gives the reference's D
    from paper_2308_07403_b200 import workloads as wl

    g = wl.er_graph(400, 0.05, 2)
    gamma = 0.2  # > 1 / rho (rho ~ 20)
    d = rb.rounded_r_distance(rb.resolvent(g, gamma, with_residual=False))
    ref = orc.run_rdist(np.asarray(g.weights), gamma)
    np.testing.assert_array_equal(d, ref)
