"""Scheduled stage-1 kernel (K1 v4, csrc/sketch_right_sched.cu) against the
CPU oracle: Y = A · Omega1^* must be bit-identical to the reference's
sem_gather_dense + fast_adjoint_right (sketch.py:362-368; _fast.pyx:23-54)
for every staging geometry the kernel picks (rows per block 1/2/4, one to
32 column chunks, 1/2/4/5/8 buckets per lane, fp32 and fp64 A, ragged m).
Inputs span 40 decades so that any change of the per-bucket summation order
shows up in the last bits."""

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


def _wide_range(m, n, seed, dtype):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n)) * 10.0 ** rng.integers(-20, 20, size=(m, n))
    return a.astype(dtype)


# (m, n, dtype, l1, k1): geometry noted per case (rb = rows per block)
SHAPES = [
    (300, 2048, np.float64, 480, 60),     # config-1 shape: 16 KB rows, rb 2, 1 chunk
    (257, 1024, np.float32, 200, 30),     # 4 KB rows, rb 4, ragged m
    (200, 16384, np.float32, 880, 110),   # config-2 shape: rb 1, 2 chunks
    (150, 8192, np.float32, 1760, 220),   # config-3 shape: rb 1, 2 buckets per lane
    (64, 30000, np.float32, 3000, 100),   # 4 chunks, 4 buckets per lane
    (100, 12000, np.float64, 700, 64),    # fp64, 3 chunks
    (3, 4096, np.float32, 64, 16),        # fewer row blocks than SMs
    (24, 65536, np.float64, 4400, 550),   # config-5 shape: 5 buckets per lane, > 4 chunks
                                          # (codes in global memory), 9 of 16 FWHT blocks stored
    (40, 50000, np.float32, 1000, 90),    # fp32 rows over 4 chunks: codes in global memory
    (9, 20000, np.float64, 6000, 80),     # 8 buckets per lane
]


@pytest.mark.parametrize("m,n,dt,l,k", SHAPES)
def test_scheduled_k1_bit_exact(P, m, n, dt, l, k):
    import torch
    from oracle import draws as D
    from oracle import randlu as O
    from paper_1601_04280_b200 import _lib
    seed = 11 + m
    dcode = _lib.SRLU_F32 if dt == np.float32 else _lib.SRLU_F64
    pad = 1 << (l - 1).bit_length()
    assert _lib.lib().srlu_k1_schedule_bytes(n, l, pad, dcode) > 0, "shape should be scheduled"
    a = _wide_range(m, n, seed, dt)
    om = P.build_composite(k, l, n, "hadamard", seed)
    y = P.apply_sketch_right(P.Matrix.from_device(torch.from_numpy(a).cuda()), om)
    ref = O.apply_sketch_right(a.astype(np.float64), D.build_composite(k, l, n, seed))
    np.testing.assert_array_equal(y.numpy(), ref)


def test_scheduled_matches_unscheduled_kernel(P, monkeypatch):
    import torch
    m, n, l, k = 500, 16384, 880, 110
    a = torch.from_numpy(_wide_range(m, n, 3, np.float32)).cuda()
    om = P.build_composite(k, l, n, "hadamard", 9)
    y1 = P.apply_sketch_right(P.Matrix.from_device(a), om).numpy()
    monkeypatch.setenv("SRLU_K1_NOSCHED", "1")
    om2 = P.build_composite(k, l, n, "hadamard", 9)
    y2 = P.apply_sketch_right(P.Matrix.from_device(a), om2).numpy()
    np.testing.assert_array_equal(y1, y2)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_scheduled_k1_non_finite_flag(P, dt):
    import torch
    m, n, l, k = 40, 2048, 300, 40
    a = np.random.default_rng(0).standard_normal((m, n)).astype(dt)
    a[37, 1999] = np.inf
    om = P.build_composite(k, l, n, "hadamard", 1)
    with pytest.raises(ValueError):
        P.apply_sketch_right(P.Matrix.from_device(torch.from_numpy(a).cuda()), om)


# unscheduled TMA kernel (k1v2): shapes the schedule does not take (rows over
# 4 chunks, l1 > 3584) and every slot count it dispatches (1, 2, 4, 5, 8)
V2_SHAPES = [
    (40, 65536, np.float64, 4400, 550),   # config-5 shape family: 5 slots, 8 KB-pad FWHT
    (33, 40000, np.float64, 3000, 100),   # 4 slots
    (20, 20000, np.float64, 1500, 64),    # 2 slots, ragged chunks
    (17, 9000, np.float64, 6000, 80),     # 8 slots
    (50, 70000, np.float32, 900, 90),     # 1 slot, fp32 rows over 4 chunks
]


@pytest.mark.parametrize("m,n,dt,l,k", V2_SHAPES)
def test_unscheduled_k1_bit_exact(P, m, n, dt, l, k, monkeypatch):
    import torch
    from oracle import draws as D
    from oracle import randlu as O
    monkeypatch.setenv("SRLU_K1_NOSCHED", "1")
    seed = 5 + m
    a = _wide_range(m, n, seed, dt)
    om = P.build_composite(k, l, n, "hadamard", seed)
    y = P.apply_sketch_right(P.Matrix.from_device(torch.from_numpy(a).cuda()), om)
    ref = O.apply_sketch_right(a.astype(np.float64), D.build_composite(k, l, n, seed))
    np.testing.assert_array_equal(y.numpy(), ref)


# TMEM-accumulator kernel (csrc/sketch_right_tmem.cu), opt-in: lanes = rows,
# bucket sums in tensor memory, 128 <= pad1 <= 1024
K1T_SHAPES = [
    (300, 2048, np.float64, 480, 60, "8"),     # one row group, fp64
    (200, 4096, np.float32, 880, 110, "28"),   # three 8-row boxes + a 4-row tail box, skew warps
    (4000, 4096, np.float32, 880, 110, "16"),  # several row blocks per CTA
    (100, 3000, np.float64, 700, 64, "32"),    # fp64, four row groups
    (257, 1024, np.float32, 200, 30, ""),      # pad 256 (64 slots per quarter), rows picked
]


@pytest.mark.parametrize("m,n,dt,l,k,rows", K1T_SHAPES)
def test_tmem_k1_bit_exact(P, m, n, dt, l, k, rows, monkeypatch):
    import torch
    from oracle import draws as D
    from oracle import randlu as O
    monkeypatch.setenv("SRLU_K1_TMEM", "1")
    if rows:
        monkeypatch.setenv("SRLU_K1T_ROWS", rows)
    seed = 23 + m
    a = _wide_range(m, n, seed, dt)
    om = P.build_composite(k, l, n, "hadamard", seed)
    y = P.apply_sketch_right(P.Matrix.from_device(torch.from_numpy(a).cuda()), om)
    ref = O.apply_sketch_right(a.astype(np.float64), D.build_composite(k, l, n, seed))
    np.testing.assert_array_equal(y.numpy(), ref)


# K1-CSR (warp per row): several pads, chunk counts and same-bucket collisions
@pytest.mark.parametrize("m,n,l,k,dens,dt", [
    (3000, 4000, 600, 64, 0.01, np.float32),     # pad 1024, two 512-point blocks
    (1500, 2500, 300, 40, 0.02, np.float64),     # pad 512, one block
    (700, 3000, 1000, 120, 0.05, np.float64),    # ~150 entries per row: several chunks, same-bucket lanes
    (900, 5000, 200, 30, 0.01, np.float32),      # pad 256
])
def test_csr_k1_bit_exact(P, m, n, l, k, dens, dt):
    from scipy.sparse import random as sprandom
    from oracle import draws as D
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(100 + m))
    a = sprandom(m, n, density=dens, format="csr", random_state=g, dtype=np.float64)
    a.data = (g.standard_normal(a.nnz) * 10.0 ** g.integers(-12, 12, size=a.nnz)).astype(dt)
    a = a.astype(dt)
    om = P.build_composite(k, l, n, "hadamard", 17)
    y = P.apply_sketch_right(P.Matrix.sparse(a), om)
    ref = O.sketch_right_rows(a.astype(np.float64), D.build_composite(k, l, n, 17))
    np.testing.assert_array_equal(y.numpy(), ref)
