"""Parity of the CUDA path (through the C ABI) with the reference.

Bit-exact: draws, the bucket plan, Y (stage-1 sketch), P, L1, both stage-2
reductions, Q.  Tolerance (north star): L and U within 1e-10 relative
(Frobenius) of the reference, ||LU - PAQ||_F within 1%.  Golden vectors
were produced by the reference itself (tests/golden/make_golden.py)."""

import hashlib
import logging

import numpy as np
import pytest

from tests.conftest import cuda_ok
from tests.golden import cases
from tests.parity import check_tail

pytestmark = pytest.mark.gpu

LU_RTOL = 1e-10


@pytest.fixture(scope="module")
def P():
    if not cuda_ok():
        pytest.skip("needs a CUDA device")
    import paper_1601_04280_b200 as pkg
    return pkg


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _np(t):
    import torch
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    if hasattr(t, "numpy"):
        return t.numpy()
    return np.asarray(t)


def _rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# --------------------------------------------------------------------------
# K0 draws


@pytest.mark.parametrize("name", list(cases.DRAW_SHAPES))
def test_device_draws_match_reference(P, golden, name):
    g = golden("draws.npz")
    k, l, n, seed = cases.DRAW_SHAPES[name]
    om = P.build_composite(k, l, n, "hadamard", seed)
    row_of = _np(om.sem.row_of).astype(np.int64)
    sign = _np(om.sem.sign)
    assert _sha(row_of) == g[name + "_row_of_sha"].item().decode()
    assert _sha(sign) == g[name + "_sign_sha"].item().decode()
    np.testing.assert_array_equal(_np(om.fast.phase), g[name + "_phase"])
    np.testing.assert_array_equal(_np(om.fast.sample_idx), g[name + "_idx"])
    assert om.fast.pad == int(g[name + "_pad"]) and om.fast.scale == float(g[name + "_scale"])


def test_draws_rejection_heavy_range(P):
    # l = 2^20 buckets: ~500 Lemire rejections in 2^21 draws; the device
    # position remapping must match numpy's sequential stream exactly
    l, n, seed = 2 ** 20, 2 ** 21, 77
    om = P.build_sem(l, n, seed)
    g = np.random.Generator(np.random.Philox(seed))
    np.testing.assert_array_equal(_np(om.row_of), g.integers(0, l, size=n))
    np.testing.assert_array_equal(_np(om.sign), (g.integers(0, 2, size=n) * 2 - 1).astype(float))


def test_sem_plan_is_stable_bucket_sort(P):
    sem = P.build_sem(97, 20000, 5)
    srt, bptr = sem.plan()
    srt, bptr = _np(srt), _np(bptr)
    row_of, sign = _np(sem.row_of), _np(sem.sign)
    src = srt & 0x7FFFFFFF
    neg = srt < 0
    assert np.array_equal(np.diff(bptr), np.bincount(row_of, minlength=97))
    for t in range(97):
        seg = src[bptr[t]:bptr[t + 1]]
        assert np.all(np.diff(seg) > 0)
        assert np.all(row_of[seg] == t)
    assert np.array_equal(neg, sign[src] < 0)


# --------------------------------------------------------------------------
# the plugin seam (_kernels) against the reference's own kernel outputs


def test_kernel_seam_matches_reference(P, golden):
    import torch
    from paper_1601_04280_b200 import _kernels as K
    g = golden("kernels.npz")
    for name, case in cases.kernel_cases().items():
        kind = case["kind"]
        if kind == "fwht":
            x = torch.tensor(case["x"], device="cuda")
            K.fwht_rows(x)
            got = x
        elif kind == "gather_dense":
            out = torch.zeros(case["out_shape"], dtype=torch.float64, device="cuda")
            K.sem_gather_dense(torch.tensor(case["a"], device="cuda"), case["row_of"],
                               case["sign"], out)
            got = out
        elif kind == "scatter_dense":
            out = torch.zeros(case["out_shape"], dtype=torch.float64, device="cuda")
            K.sem_scatter_dense(torch.tensor(case["a"], device="cuda"), case["row_of"],
                                case["sign"], out)
            got = out
        else:
            sp = case["csc"]
            out = torch.zeros(case["out_shape"], dtype=torch.float64, device="cuda")
            fn = K.sem_gather_csc if kind == "gather_csc" else K.sem_scatter_csc
            fn(torch.tensor(sp.data), torch.tensor(sp.indices), torch.tensor(sp.indptr),
               case["row_of"], case["sign"], out)
            got = out
        np.testing.assert_array_equal(_np(got), g[name], err_msg=name)


# --------------------------------------------------------------------------
# K2 / K5 pivoted LUs against the reference's factor.py


def test_factor_matches_reference(P, golden):
    g = golden("factor.npz")
    for name, b in cases.factor_cases().items():
        if b.shape[0] >= b.shape[1]:
            r = P.lu_row_pivot(b)
            np.testing.assert_array_equal(r.P.indices, g[name + "_row_P"], err_msg=name)
            np.testing.assert_array_equal(r.L.numpy(), g[name + "_row_L"], err_msg=name)
            np.testing.assert_array_equal(r.U.numpy(), g[name + "_row_U"], err_msg=name)
        bt = b.T if b.shape[0] >= b.shape[1] else b
        c = P.lu_col_pivot(bt)
        np.testing.assert_array_equal(c.Q.indices, g[name + "_col_Q"], err_msg=name)
        np.testing.assert_array_equal(c.L.numpy(), g[name + "_col_L"], err_msg=name)
        np.testing.assert_array_equal(c.U.numpy(), g[name + "_col_U"], err_msg=name)


@pytest.mark.parametrize("m,k,seed,ints", [(20000, 200, 1, False), (6000, 150, 2, True),
                                           (3001, 97, 3, False), (40000, 64, 4, False)])
@pytest.mark.parametrize("gpanel", ["0", "1"])
def test_lu_row_pivot_panels_bit_exact(P, m, k, seed, ints, gpanel, monkeypatch):
    """Sizes that force several panels + deferred trailing updates; gpanel=1
    forces the grid kernel's in-place (L2) panel variant used for tall inputs."""
    monkeypatch.setenv("SRLU_LU_GPANEL", gpanel)
    monkeypatch.setenv("SRLU_LU_NO_HYBRID", gpanel)
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(seed))
    b = g.integers(-3, 4, size=(m, k)).astype(np.float64) if ints else g.standard_normal((m, k))
    perm, lo, up = O.lu_row_pivot(b)
    r = P.lu_row_pivot(b)
    np.testing.assert_array_equal(r.P.indices, perm)
    np.testing.assert_array_equal(r.L.numpy(), lo)
    np.testing.assert_array_equal(r.U.numpy(), up)


@pytest.mark.parametrize("k,n,seed", [(150, 30000, 5), (97, 5003, 6), (40, 100000, 7)])
@pytest.mark.parametrize("gpanel", ["0", "1"])
def test_lu_col_pivot_panels_bit_exact(P, k, n, seed, gpanel, monkeypatch):
    monkeypatch.setenv("SRLU_LU_GPANEL", gpanel)
    monkeypatch.setenv("SRLU_LU_NO_HYBRID", gpanel)
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(seed))
    c = g.standard_normal((k, n))
    q, lo, up = O.lu_col_pivot(c)
    r = P.lu_col_pivot(c)
    np.testing.assert_array_equal(r.Q.indices, q)
    np.testing.assert_array_equal(r.L.numpy(), lo)
    np.testing.assert_array_equal(r.U.numpy(), up)


@pytest.mark.parametrize("m,k,seed", [(16384, 110, 8), (6000, 150, 2), (2048, 60, 9),
                                      (8192, 220, 10), (4096, 128, 11), (2048, 300, 12)])
def test_lu_cluster_and_grid_variants_agree(P, m, k, seed, monkeypatch):
    """The LU kernels on one input: hybrid (default for m <= 16384), the
    148-CTA grid kernel (SRLU_LU_NO_HYBRID=1) and its in-place-panel variant
    (+ SRLU_LU_GPANEL=1) must give the oracle's P, L, U (row) and Q, L, U (col)."""
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(seed))
    b = g.standard_normal((m, k))
    perm, lo, up = O.lu_row_pivot(b)
    q, lo2, up2 = O.lu_col_pivot(b.T.copy())
    for mode in ("hybrid", "grid", "gpanel"):
        no_cluster = mode
        monkeypatch.setenv("SRLU_LU_NO_HYBRID", "0" if mode == "hybrid" else "1")
        monkeypatch.setenv("SRLU_LU_GPANEL", "1" if mode == "gpanel" else "0")
        r = P.lu_row_pivot(b)
        np.testing.assert_array_equal(r.P.indices, perm, err_msg=no_cluster)
        np.testing.assert_array_equal(r.L.numpy(), lo, err_msg=no_cluster)
        np.testing.assert_array_equal(r.U.numpy(), up, err_msg=no_cluster)
        c = P.lu_col_pivot(b.T.copy())
        np.testing.assert_array_equal(c.Q.indices, q, err_msg=no_cluster)
        np.testing.assert_array_equal(c.L.numpy(), lo2, err_msg=no_cluster)
        np.testing.assert_array_equal(c.U.numpy(), up2, err_msg=no_cluster)


def test_lu_low_rank_threshold_path(P):
    """Exactly low rank: later pivots fall under PIVOT_RTOL*||B||_F."""
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(11))
    b = g.standard_normal((5000, 6)) @ g.standard_normal((6, 40))
    perm, lo, up = O.lu_row_pivot(b)
    r = P.lu_row_pivot(b)
    np.testing.assert_array_equal(r.P.indices, perm)
    np.testing.assert_array_equal(r.L.numpy(), lo)
    q, lo2, up2 = O.lu_col_pivot(b[:40].T.copy())
    c = P.lu_col_pivot(b[:40].T.copy())
    np.testing.assert_array_equal(c.Q.indices, q)
    np.testing.assert_array_equal(c.L.numpy(), lo2)


# --------------------------------------------------------------------------
# the whole path against the reference's outputs (golden)

PIPES = ["small_dense", "ragged", "sparse", "zero", "lowrank_resample", "tall_f32",
         "sparse_wide", "cfg1"]


def _input(P, a, as_f32=False):
    import torch
    if hasattr(a, "tocsr"):
        return P.Matrix.sparse(a)
    t = torch.tensor(np.ascontiguousarray(a), device="cuda")
    if as_f32:
        t = t.float()
    return P.Matrix.from_device(t)


@pytest.mark.parametrize("name", PIPES)
def test_pipeline_matches_reference(P, golden, name):
    g = golden(f"pipe_{name}.npz")
    a, prm = cases.pipeline_cases()[name]
    # tall_f32 holds float32-representable values: feed it as float32 storage
    mat = _input(P, a, as_f32=(name == "tall_f32"))
    res = P.sparse_randomized_lu(mat, P.RandLuParams(**prm), keep=True)
    ex = res.extras
    assert res.attempt == int(g["attempt"])
    np.testing.assert_array_equal(_np(ex["Y"]), g["Y"])
    np.testing.assert_array_equal(res.P.indices, g["P"])
    if "L1" in g:
        np.testing.assert_array_equal(_np(ex["L1"]), g["L1"])
    np.testing.assert_array_equal(_np(ex["red_l"]), g["red_l"])
    np.testing.assert_array_equal(_np(ex["red_a"]), g["red_a"])
    assert _rel(_np(ex["core"]), g["core"]) <= 1e-12
    l1 = g["L1"] if "L1" in g else _np(ex["L1"])
    check_tail(res.Q.indices, res.L.numpy(), res.U.numpy(), g["Q"], g["L"], g["U"], g["core"],
               g["red_l"], g["red_a"], l1)
    err = P.approximation_error(mat, res)
    want = float(g["err"])
    anorm = np.linalg.norm(a.toarray() if hasattr(a, "toarray") else a)
    assert abs(err - want) <= 0.01 * want + 1e-12 * anorm
    assert set(res.elapsed) == {"sketch1", "lu1", "sketch2", "pinv", "lu2", "total"}


def test_resample_warnings(P, caplog):
    a, prm = cases.pipeline_cases()["lowrank_resample"]
    with caplog.at_level(logging.WARNING, logger="paper_1601_04280_b200.randlu"):
        res = P.sparse_randomized_lu(a, P.RandLuParams(**prm))
    assert res.attempt == 2
    assert sum("resampling" in r.message for r in caplog.records) == 2


def test_determinism_bit_identical(P):
    a, prm = cases.pipeline_cases()["small_dense"]
    r1 = P.sparse_randomized_lu(a, P.RandLuParams(**prm))
    r2 = P.sparse_randomized_lu(a, P.RandLuParams(**prm))
    assert np.array_equal(r1.P.indices, r2.P.indices)
    assert np.array_equal(r1.Q.indices, r2.Q.indices)
    np.testing.assert_array_equal(r1.L.numpy(), r2.L.numpy())
    np.testing.assert_array_equal(r1.U.numpy(), r2.U.numpy())


def test_zero_matrix_zero_error(P):
    a = np.zeros((60, 50))
    res = P.sparse_randomized_lu(a, P.RandLuParams(r=2, k1=3, l1=20, k2=4, l2=48, seed=1))
    assert P.approximation_error(a, res) == 0.0
    assert np.all(res.U.numpy() == 0.0)


def test_non_finite_rejected(P):
    import torch
    a = torch.randn(200, 150, device="cuda", dtype=torch.float64)
    a[17, 33] = float("nan")
    with pytest.raises(ValueError, match="finite"):
        P.sparse_randomized_lu(P.Matrix.from_device(a), P.default_params(5, 200, 150))
    a[17, 33] = float("inf")
    with pytest.raises(ValueError, match="finite"):
        P.sparse_randomized_lu(P.Matrix.from_device(a), P.default_params(5, 200, 150))


def test_params_checked_against_matrix(P):
    with pytest.raises(P.ParameterError):
        P.sparse_randomized_lu(np.zeros((30, 30)), P.RandLuParams(r=2, k1=3, l1=40, k2=4, l2=20))


def test_exact_rank_recovery(P):
    from tests.golden.cases import gen_rank_noise
    for seed in range(3):
        a = gen_rank_noise(300, 300, 10, 0.0, seed)
        res = P.sparse_randomized_lu(a, P.default_params(10, 300, 300, seed=100 + seed))
        assert P.approximation_error(a, res) <= 1e-8 * np.linalg.norm(a)


# --------------------------------------------------------------------------
# BASELINE config 2 at full size against the CPU oracle (same fp32 input)


@pytest.mark.slow
def test_config2_full_size_vs_oracle(P):
    import torch
    from threadpoolctl import threadpool_limits
    from oracle import randlu as O
    from bench import gen_config
    a, prm = gen_config(2)
    res = P.sparse_randomized_lu(P.Matrix.from_device(a), P.RandLuParams(**prm), keep=True)
    host = a.double().cpu().numpy()
    with threadpool_limits(8):
        ref = O.sparse_randomized_lu(host, prm, keep=True)
    np.testing.assert_array_equal(_np(res.extras["Y"]), ref["Y"])
    np.testing.assert_array_equal(res.P.indices, ref["P"])
    np.testing.assert_array_equal(_np(res.extras["red_a"]), ref["red_a"])
    check_tail(res.Q.indices, res.L.numpy(), res.U.numpy(), ref["Q"], ref["L"], ref["U"],
               ref["core"], ref["red_l"], ref["red_a"], ref["L1"])


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_csr_long_columns_bit_exact(P, dt):
    """Columns longer than the 2048-entry fast path (second launch) stay exact
    (fp32 values: the compact 8-byte entries)."""
    from scipy.sparse import csr_array
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(31))
    m, n = 6000, 300
    d = g.standard_normal((m, n))
    d[g.random((m, n)) < 0.97] = 0.0
    d[g.random(m) < 0.6, 7] = g.standard_normal(1)[0]      # ~3600 entries in column 7
    d[:, 11] = g.standard_normal(m)                          # dense column 11
    d = d.astype(dt)
    prm = dict(r=6, k1=14, l1=56, k2=22, l2=88, seed=5)
    res = P.sparse_randomized_lu(P.Matrix.sparse(csr_array(d)), P.RandLuParams(**prm), keep=True)
    ref = O.sparse_randomized_lu(csr_array(d), prm, keep=True)
    np.testing.assert_array_equal(_np(res.extras["Y"]), ref["Y"])
    np.testing.assert_array_equal(res.P.indices, ref["P"])
    np.testing.assert_array_equal(_np(res.extras["red_a"]), ref["red_a"])


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_csr_very_long_columns_bit_exact(P, dt):
    """Columns far beyond one CTA's 8192-entry sort (50k entries, a dense
    60k column): bucket-range passes, bit-exact (_fast.pyx:81-90 order)."""
    from scipy.sparse import csr_array
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(41))
    m, n = 60000, 200
    d = g.standard_normal((m, n))
    d[g.random((m, n)) < 0.995] = 0.0
    d[g.permutation(m)[:50000], 5] = g.standard_normal(50000)   # a 50k-nnz column
    d[:, 9] = g.standard_normal(m)                               # a dense column
    d = d.astype(dt)
    prm = dict(r=6, k1=14, l1=56, k2=22, l2=88, seed=5)
    res = P.sparse_randomized_lu(P.Matrix.sparse(csr_array(d)), P.RandLuParams(**prm), keep=True)
    ref = O.sparse_randomized_lu(csr_array(d), prm, keep=True)
    np.testing.assert_array_equal(_np(res.extras["Y"]), ref["Y"])
    np.testing.assert_array_equal(res.P.indices, ref["P"])
    np.testing.assert_array_equal(_np(res.extras["red_a"]), ref["red_a"])


def test_csr_oversized_bucket_group_bit_exact(P):
    """4 stage-2 buckets and a dense 40k column: ~10k entries of one column
    in one bucket (> 8192) are folded in ascending-q chunks with the running
    sum carried over — still the reference's sequential sum."""
    from scipy.sparse import csr_array
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(43))
    m, n = 40000, 24
    d = g.standard_normal((m, n)) * np.exp2(g.integers(-20, 20, size=(m, n)))
    d[g.random((m, n)) < 0.9] = 0.0
    d[:, 3] = g.standard_normal(m)
    prm = dict(r=1, k1=2, l1=8, k2=3, l2=4, seed=2)
    res = P.sparse_randomized_lu(P.Matrix.sparse(csr_array(d)), P.RandLuParams(**prm), keep=True)
    ref = O.sparse_randomized_lu(csr_array(d), prm, keep=True)
    np.testing.assert_array_equal(res.P.indices, ref["P"])
    np.testing.assert_array_equal(_np(res.extras["red_a"]), ref["red_a"])


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_csr_crowded_buckets_bit_exact(P, dt):
    """Few stage-2 buckets, ~1600 entries per column: long same-bucket runs whose
    fold order (ascending PA row) matters; values span many binades."""
    from scipy.sparse import csr_array
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(77))
    m, n = 20000, 64
    d = g.standard_normal((m, n)) * np.exp2(g.integers(-30, 30, size=(m, n)))
    d[g.random((m, n)) < 0.92] = 0.0
    d = d.astype(dt)
    prm = dict(r=4, k1=8, l1=40, k2=12, l2=24, seed=3)
    res = P.sparse_randomized_lu(P.Matrix.sparse(csr_array(d)), P.RandLuParams(**prm), keep=True)
    ref = O.sparse_randomized_lu(csr_array(d), prm, keep=True)
    np.testing.assert_array_equal(_np(res.extras["Y"]), ref["Y"])
    np.testing.assert_array_equal(res.P.indices, ref["P"])
    np.testing.assert_array_equal(_np(res.extras["red_a"]), ref["red_a"])


@pytest.mark.parametrize("n,dt", [(301, np.float32), (299, np.float64)])
def test_stage1_unaligned_rows_fused_call(P, n, dt):
    """Rows whose pitch is not a multiple of 16 bytes take the unscheduled K1
    inside the one-call stage 1 (srlu_composite_sketch_right_dense without a
    schedule): Y and P still bit-exact against the oracle."""
    import torch
    from oracle import randlu as O
    rng = np.random.default_rng(n)
    a = (rng.standard_normal((400, 12)) @ rng.standard_normal((12, n))
         + 1e-3 * rng.standard_normal((400, n))).astype(dt)
    prm = dict(r=12, k1=20, l1=80, k2=28, l2=112, seed=3)
    res = P.sparse_randomized_lu(P.Matrix.from_device(torch.from_numpy(a).cuda()),
                                 P.RandLuParams(**prm), keep=True)
    ref = O.sparse_randomized_lu(a.astype(np.float64), prm, keep=True)
    np.testing.assert_array_equal(res.extras["Y"].cpu().numpy(), ref["Y"])
    np.testing.assert_array_equal(res.P.indices, ref["P"])


# --------------------------------------------------------------------------
# round-2 code paths behind knobs: every variant must stay bit-exact


@pytest.mark.parametrize("mode", ["row", "col"])
@pytest.mark.parametrize("gpanel", ["0", "1"])
def test_lu_two_level_trailing_update_bit_exact(P, mode, gpanel, monkeypatch):
    """Grid LU with the opt-in outer-block (two-level) trailing update, for
    the shared-memory panel and the L2 panel: same P/Q, L, U bits."""
    monkeypatch.setenv("SRLU_LU_B2", "1")
    monkeypatch.setenv("SRLU_LU_NO_HYBRID", "1")
    monkeypatch.setenv("SRLU_LU_GPANEL", gpanel)
    monkeypatch.setenv("SRLU_LU_MAX_GRID", "8")   # many rows per CTA: narrow panels, b2 = 4 b
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(77))
    if mode == "row":
        b = g.standard_normal((30000, 150))
        b[:, 40:44] = b[:, :4] @ g.standard_normal((4, 4))   # dependent columns: threshold path
        perm, lo, up = O.lu_row_pivot(b)
        r = P.lu_row_pivot(b)
        np.testing.assert_array_equal(r.P.indices, perm)
        np.testing.assert_array_equal(r.L.numpy(), lo)
        np.testing.assert_array_equal(r.U.numpy(), up)
    else:
        c = g.standard_normal((120, 25000))
        q, lo, up = O.lu_col_pivot(c)
        r = P.lu_col_pivot(c)
        np.testing.assert_array_equal(r.Q.indices, q)
        np.testing.assert_array_equal(r.L.numpy(), lo)
        np.testing.assert_array_equal(r.U.numpy(), up)


def test_lu_hybrid_without_cooperative_launch_bit_exact(P, monkeypatch):
    """The hybrid LU launched without the cooperative attribute (what runs
    under ncu): own grid barrier, same result."""
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(78))
    b = g.standard_normal((9000, 96))
    perm, lo, up = O.lu_row_pivot(b)
    monkeypatch.setenv("SRLU_LU_NOCOOP", "1")
    r = P.lu_row_pivot(b)
    np.testing.assert_array_equal(r.P.indices, perm)
    np.testing.assert_array_equal(r.L.numpy(), lo)
    np.testing.assert_array_equal(r.U.numpy(), up)


@pytest.mark.parametrize("knob", [None, ("SRLU_CSR_BANDS", "0"), ("SRLU_CSR_BANDFILL", "1")])
def test_csr_wide_matrix_bit_exact(P, knob, monkeypatch):
    """n >= 8192 columns: banded shared-memory column count, tiled column scan
    and absolute fill cursors (default); the global-atomic count and the
    banded fill behind their knobs."""
    if knob:
        monkeypatch.setenv(*knob)
    from scipy.sparse import random as sprandom
    from oracle import randlu as O
    g = np.random.Generator(np.random.Philox(79))
    m, n = 5000, 9000
    a = sprandom(m, n, density=0.004, format="csr", random_state=g, dtype=np.float64)
    a.data = g.standard_normal(a.nnz)
    prm = dict(r=8, k1=16, l1=64, k2=24, l2=96, seed=3)
    res = P.sparse_randomized_lu(P.Matrix.sparse(a), P.RandLuParams(**prm), keep=True)
    ref = O.sparse_randomized_lu(a, prm, keep=True)
    np.testing.assert_array_equal(_np(res.extras["Y"]), ref["Y"])
    np.testing.assert_array_equal(res.P.indices, ref["P"])
    np.testing.assert_array_equal(_np(res.extras["red_a"]), ref["red_a"])


def test_sketch_cache_reuses_draws_bit_exact(P):
    """Opt-in sketch cache: the second decomposition with the
    same parameters reuses the draws / plan / K1 schedule and returns the
    same bits; a different seed misses."""
    import torch
    g = np.random.Generator(np.random.Philox(5))
    a = torch.from_numpy(g.standard_normal((900, 700))).cuda()
    prm = dict(r=10, k1=18, l1=72, k2=26, l2=104, seed=4)
    base = P.sparse_randomized_lu(P.Matrix.from_device(a), P.RandLuParams(**prm))
    P.set_sketch_cache(True)
    try:
        r1 = P.sparse_randomized_lu(P.Matrix.from_device(a), P.RandLuParams(**prm))
        s1 = P.sketch_cache_stats()
        r2 = P.sparse_randomized_lu(P.Matrix.from_device(a), P.RandLuParams(**prm))
        s2 = P.sketch_cache_stats()
        assert s1["misses"] >= 2 and s2["hits"] >= s1["hits"] + 2 and s2["misses"] == s1["misses"]
        for r in (r1, r2):
            np.testing.assert_array_equal(r.P.indices, base.P.indices)
            np.testing.assert_array_equal(r.Q.indices, base.Q.indices)
            np.testing.assert_array_equal(r.L.numpy(), base.L.numpy())
            np.testing.assert_array_equal(r.U.numpy(), base.U.numpy())
        P.sparse_randomized_lu(P.Matrix.from_device(a), P.RandLuParams(**dict(prm, seed=6)))
        assert P.sketch_cache_stats()["misses"] > s2["misses"]
    finally:
        P.set_sketch_cache(False)
    assert P.sketch_cache_stats()["entries"] == 0
