"""Stage-2 projection (K3 = K3a bucket sums + K3b column FWHT/sample)
against the CPU oracle (sketch.py:371-378, _fast.pyx:71-78 + 23-41):
bit-exact at small shapes covering odd column counts (scalar staging
path), partial 32-column tiles, pad2 128..1024 and l2 < pad2."""

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


@pytest.mark.parametrize("m,n,l,k", [(300, 18, 104, 26), (300, 240, 104, 26),
                                     (2000, 64, 104, 26), (600, 18, 472, 118),
                                     (500, 35, 104, 26), (3000, 97, 900, 200),
                                     (3000, 37, 2232, 558)])  # config-5 pad2 4096: K3b v2, 4 columns per CTA
@pytest.mark.parametrize("v2", [False, True])
def test_sketch_left_bit_exact(P, monkeypatch, m, n, l, k, v2):
    from oracle import draws as D
    from oracle import randlu as O
    if v2:
        monkeypatch.setenv("SRLU_K3B_V2", "1")
    a = np.random.default_rng(m + n).standard_normal((m, n))
    om = P.build_composite(k, l, m, "hadamard", 5)
    got = P.apply_sketch_left(om, P.Matrix(a)).numpy()
    ref = O.apply_sketch_left(D.build_composite(k, l, m, 5), a)
    np.testing.assert_array_equal(got, ref)
