"""Dense-Gaussian baseline (gaussian_randomized_lu, reference
randlu.py:184-205, 216-219) against fixtures made by
the reference itself (tests/golden/make_golden_gauss.py).  The products are
cuBLAS here and OpenBLAS there, so: P identical, Q identical on the signal
pivots (the first r; later ones are chosen among noise-level values), the
signal part of L and U within 1e-8 relative, ||LU - PAQ||_F within 1%."""

import os

import numpy as np
import pytest

from tests.conftest import cuda_ok
from tests.golden import cases
from tests.golden.make_golden_gauss import CASES

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def P():
    if not cuda_ok():
        pytest.skip("needs a CUDA device")
    import paper_1601_04280_b200 as pkg
    return pkg


@pytest.mark.parametrize("name", sorted(CASES))
def test_gaussian_baseline_matches_reference(P, name):
    from scipy.sparse import csc_array
    g = np.load(os.path.join(HERE, "golden", "gauss.npz"))
    c = CASES[name]
    a = cases.gen_rank_noise(c["m"], c["n"], c["r"], c["noise"], c["seed"])
    if "density" in c:
        a[np.random.default_rng(c["seed"]).random(a.shape) >= c["density"]] = 0.0
        mat = P.Matrix.sparse(csc_array(a))
    else:
        mat = P.Matrix(a)
    r, seed = c["prm"]
    res = P.gaussian_randomized_lu(mat, P.default_params(r, c["m"], c["n"], seed=seed))
    np.testing.assert_array_equal(res.P.indices, g[name + "_P"])
    np.testing.assert_array_equal(res.Q.indices[:r], g[name + "_Q"][:r])
    L, U = res.L.numpy(), res.U.numpy()
    gl, gu = g[name + "_L"], g[name + "_U"]
    assert np.abs(L[:, :r] - gl[:, :r]).max() <= 1e-8 * np.abs(gl[:, :r]).max()
    assert np.abs(U[:r] - gu[:r]).max() <= 1e-8 * np.abs(gu[:r]).max()
    err = P.approximation_error(mat, res)
    ref = float(g[name + "_err"])
    assert abs(err - ref) <= 0.01 * ref, (err, ref)
