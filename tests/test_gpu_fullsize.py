"""Parity at the BASELINE configs' full sizes (3: 262144 x 8192 fp32 dense,
4: 1048576 x 65536 CSR, 5: 65536 x 65536 fp64), where the CPU oracle cannot run the whole pipeline
in test time.  Size-independent properties instead:

* Y = A . Omega1^* row by row: every row of Y depends only on the same row of
  A, so sampled rows are compared bit-for-bit with the oracle's sketch of
  those rows (sketch.py:362-368);
* LU(Y) = GEPP (factor.py:49-77): |L1| <= 1 with a unit diagonal (the
  pivot is the column maximum), P a permutation, and P.Y = L1.U1 on sampled
  rows to round-off (U1 from the leading rows);
* Omega2 . (P A) column by column: sampled columns are compared bit-for-bit
  with the oracle's left sketch of the same columns of P A (given the
  device's P, sketch.py:371-378);
* LU(core) = GE with column pivoting (factor.py:80-109): |U[i, j]| <=
  |U[i, i]| for j >= i, Q a permutation, L~ unit lower triangular.
"""

import numpy as np
import pytest

from tests.conftest import cuda_ok

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not cuda_ok():
        pytest.skip("needs a CUDA device")
    import paper_1601_04280_b200 as pkg
    return pkg


def _np(t):
    return t.detach().cpu().numpy()


def _host_csr(a, shape):
    from scipy.sparse import csr_array
    indptr, indices, values = (_np(t) for t in a)
    return csr_array((values.astype(np.float64), indices, indptr), shape=shape)


@pytest.mark.parametrize("config", [3, 4, 5])
def test_full_size_properties(P, config):
    import scipy.linalg as sla
    import torch
    from bench import CONFIGS, as_matrix, gen_config
    from oracle import draws as D
    from oracle import randlu as O

    cfg = CONFIGS[config]
    m, n = cfg["m"], cfg["n"]
    a, prm = gen_config(config)
    res = P.sparse_randomized_lu(as_matrix(P, a, (m, n)), P.RandLuParams(**prm), keep=True)
    k1, k2 = prm["k1"], prm["k2"]
    seed = prm["seed"] + 2 * res.attempt
    om1 = D.build_composite(k1, prm["l1"], n, seed)
    om2 = D.build_composite(k2, prm["l2"], m, seed + 1)
    rng = np.random.default_rng(config)
    rows = np.sort(rng.choice(m, 256, replace=False))
    cols = np.sort(rng.choice(n, 32, replace=False))
    sparse = isinstance(a, tuple)
    host = _host_csr(a, (m, n)) if sparse else None

    # --- stage 1, bit-exact on sampled rows
    a_rows = host[rows].tocsc() if sparse else _np(a[torch.from_numpy(rows).cuda()]).astype(np.float64)
    y_ref = O.apply_sketch_right(O.as_matrix(a_rows), om1)
    y = _np(res.extras["Y"])
    np.testing.assert_array_equal(y[rows], y_ref)

    # --- LU(Y): GEPP properties
    perm = res.P.indices
    assert np.array_equal(np.sort(perm), np.arange(m))
    l1 = _np(res.extras["L1"])
    assert np.all(np.abs(l1) <= 1.0)
    assert np.all(np.diag(l1[:k1]) == 1.0)
    assert np.all(np.triu(l1[:k1], 1) == 0.0)
    py = y[perm]
    u1 = sla.solve_triangular(l1[:k1], py[:k1], lower=True, unit_diagonal=True)
    resid = np.abs(py[rows] - l1[rows] @ u1).max() / np.abs(y).max()
    assert resid < 1e-10, resid

    # --- Omega2 . (P A), bit-exact on sampled columns
    if sparse:
        a_cols = host.tocsc()[:, cols].toarray()
    else:
        a_cols = _np(a[:, torch.from_numpy(cols).cuda()]).astype(np.float64)
    red_ref = O.apply_sketch_left(om2, np.asfortranarray(a_cols[perm]))
    red = _np(res.extras["red_a"])  # k2 x n
    np.testing.assert_array_equal(red[:, cols], red_ref)

    # --- LU(core): column-pivoting properties
    q = res.Q.indices
    assert np.array_equal(np.sort(q), np.arange(n))
    u = res.U.numpy()
    lt = _np(res.extras["Lt"])
    for i in range(k1):
        piv = abs(u[i, i])
        assert np.all(np.abs(u[i, i:]) <= piv), i
        assert np.all(u[i, :i] == 0.0)
    lt_h = lt if lt.shape == (k1, k1) else lt.T
    assert np.all(np.diag(lt_h) == 1.0)
    assert np.all(np.triu(lt_h, 1) == 0.0) or np.all(np.tril(lt_h, -1) == 0.0)
    err = P.approximation_error(as_matrix(P, a, (m, n)), res)
    assert np.isfinite(err)
