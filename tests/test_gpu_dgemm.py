"""FP64 tensor-core GEMM (libsrlu srlu_dgemm_ex, DMMA) and the fused
approximation error K7 (srlu_lu_error_dense / _csr).

The GEMMs replace the reference's BLAS matmul (randlu.py:267 core,
randlu.py:272 L = L1 L~; matrix.py:219-230).  A different BLAS orders the
k-sums differently, so the criterion is the fp64 forward-error bound of a
dot product: |C - C_exact| <= 2 K u |A| |B| elementwise (u = 2^-53), with
C_exact from an extended-precision (long double) product on the host.
K7 (randlu.py:279-302) is checked against the oracle's column-block
restatement at 1e-12 relative.
"""

import numpy as np
import pytest

from tests.conftest import cuda_ok

pytestmark = pytest.mark.gpu

U64 = 2.0 ** -53


@pytest.fixture(scope="module")
def P():
    if not cuda_ok():
        pytest.skip("needs a CUDA device")
    import paper_1601_04280_b200 as pkg
    return pkg


def _exact(a, b):
    return (a.astype(np.longdouble) @ b.astype(np.longdouble))


def _check_bound(c, a, b):
    k = a.shape[1]
    ex = _exact(a, b)
    bound = 2.0 * max(k, 1) * U64 * (np.abs(a) @ np.abs(b)) + 1e-300
    err = np.abs(c.astype(np.longdouble) - ex)
    assert np.all(err <= bound), float(np.max(err / bound))


@pytest.mark.parametrize("m,n,k", [
    (1, 1, 1), (7, 5, 3), (129, 65, 17), (300, 110, 118),   # config-2 core shape (small m)
    (1000, 550, 558), (4096, 220, 220), (2000, 120, 120),  # config 5 / 3 / 4 shapes
    (513, 37, 41), (255, 129, 33), (16384, 110, 118),
])
@pytest.mark.parametrize("tile", ["", "0", "1", "2", "3"])
def test_dgemm_matches_exact(P, monkeypatch, m, n, k, tile):
    import torch
    from paper_1601_04280_b200.factor import dgemm
    if tile:
        monkeypatch.setenv("SRLU_DGEMM_TILE", tile)
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((k, n))
    c = dgemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    _check_bound(c, a, b)


@pytest.mark.parametrize("m,k", [(5000, 110), (3000, 550), (777, 33), (64, 64)])
def test_dgemm_lower_triangular_b(P, m, k):
    """L = L1 . L~ with L~ unit lower triangular: the zero blocks above the
    diagonal are skipped; same bound as the full product."""
    import torch
    from paper_1601_04280_b200.factor import dgemm
    rng = np.random.default_rng(m + k)
    a = rng.uniform(-1, 1, (m, k))
    b = np.tril(rng.uniform(-1, 1, (k, k)), -1) + np.eye(k)
    c = dgemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), b_lower=True)
    _check_bound(c.cpu().numpy(), a, b)


def test_dgemm_strided_and_unaligned(P):
    """Leading dimensions larger than the width, odd widths (8-byte copy path)."""
    import torch
    from paper_1601_04280_b200.factor import dgemm
    rng = np.random.default_rng(3)
    big_a = torch.from_numpy(rng.standard_normal((400, 71))).cuda()
    big_b = torch.from_numpy(rng.standard_normal((61, 90))).cuda()
    a = big_a[:, 1:62]          # 400 x 61, ld 71, 8-byte offset
    b = big_b[:, :77]           # 61 x 77, ld 90
    out = torch.zeros(400, 80, dtype=torch.float64, device="cuda")
    dgemm(a, b, out=out[:, :77])
    _check_bound(out[:, :77].cpu().numpy(), a.cpu().numpy(), b.cpu().numpy())
    assert float(out[:, 77:].abs().max()) == 0.0


def test_dgemm_launches_dmma_kernel(P):
    """The product path is the libsrlu DMMA kernel (not cuBLAS)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_1601_04280_b200.factor import dgemm
    a = torch.randn(4096, 118, dtype=torch.float64, device="cuda")
    b = torch.randn(118, 110, dtype=torch.float64, device="cuda")
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        dgemm(a, b)
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    assert any("gemm_kernel" in x and "dmma" in x for x in names), names
    assert not any("cutlass" in x or "gemm_sm" in x.lower() for x in names), names


def _err_ref(a, perm, q, l, u):
    """randlu.py:279-302 restated (oracle.randlu.approximation_error)."""
    from oracle import randlu as O
    return O.approximation_error(a, dict(P=perm, Q=q, L=l, U=u))


@pytest.mark.parametrize("m,n,k", [(300, 200, 20), (1000, 700, 64), (777, 333, 37),
                                   (129, 2000, 110)])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_lu_error_dense_matches_oracle(P, m, n, k, dt):
    import torch
    rng = np.random.default_rng(m + n + k)
    a = rng.standard_normal((m, n))
    if dt == "f32":
        a = a.astype(np.float32).astype(np.float64)
    perm = rng.permutation(m)
    q = rng.permutation(n)
    l = rng.standard_normal((m, k))
    u = rng.standard_normal((k, n))
    ta = torch.from_numpy(a.astype(np.float32 if dt == "f32" else np.float64)).cuda()
    res = P.RandLuResult(P=P.Permutation(perm), Q=P.Permutation(q),
                         L=P.Matrix.from_device(torch.from_numpy(l).cuda()),
                         U=P.Matrix.from_device(torch.from_numpy(u).cuda()))
    got = P.approximation_error(P.Matrix.from_device(ta), res)
    ref = _err_ref(a, perm, q, l, u)
    assert abs(got - ref) <= 1e-12 * ref, (got, ref)


@pytest.mark.parametrize("m,n,k,dens", [(500, 300, 12, 0.02), (1200, 700, 33, 0.01),
                                        (300, 5000, 64, 0.003)])
def test_lu_error_csr_matches_oracle(P, m, n, k, dens):
    import scipy.sparse as sp
    import torch
    rng = np.random.default_rng(m + n)
    a = sp.random(m, n, density=dens, random_state=rng, format="csr", dtype=np.float64)
    perm = rng.permutation(m)
    q = rng.permutation(n)
    # near-exact factors: small residual, so cancellation would show
    l = rng.standard_normal((m, k))
    u = rng.standard_normal((k, n)) * 1e-3
    res = P.RandLuResult(P=P.Permutation(perm), Q=P.Permutation(q),
                         L=P.Matrix.from_device(torch.from_numpy(l).cuda()),
                         U=P.Matrix.from_device(torch.from_numpy(u).cuda()))
    got = P.approximation_error(P.Matrix(a), res)
    ref = _err_ref(a, perm, q, l, u)
    assert abs(got - ref) <= 1e-12 * ref, (got, ref)
    # and the zero residual of exact factors of a sparse matrix
    z = sp.csr_array((m, n))
    res0 = P.RandLuResult(P=P.Permutation(np.arange(m)), Q=P.Permutation(np.arange(n)),
                          L=P.Matrix.from_device(torch.zeros(m, k, dtype=torch.float64,
                                                             device="cuda")),
                          U=P.Matrix.from_device(torch.zeros(k, n, dtype=torch.float64,
                                                             device="cuda")))
    assert P.approximation_error(P.Matrix(z), res0) == 0.0
