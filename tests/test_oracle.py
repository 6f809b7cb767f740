"""Pin the CPU oracle to the reference: every golden vector the reference
produced (tests/golden/make_golden.py) must be reproduced bit-for-bit,
plus the reference's own known-answer tests (cited inline)."""

import hashlib
import math

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

from oracle import draws, randlu as O
from tests.golden import cases


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --------------------------------------------------------------------------
# draws (sketch.py:103-114, 214-235, 269-278)


@pytest.mark.parametrize("name", list(cases.DRAW_SHAPES))
def test_draws_match_reference(name, golden):
    g = golden("draws.npz")
    k, l, n, seed = cases.DRAW_SHAPES[name]
    om = draws.build_composite(k, l, n, seed)
    assert _sha(om["row_of"].astype(np.int64)) == g[name + "_row_of_sha"].item().decode()
    assert _sha(om["sign"]) == g[name + "_sign_sha"].item().decode()
    np.testing.assert_array_equal(om["phase"], g[name + "_phase"])
    np.testing.assert_array_equal(om["sample_idx"], g[name + "_idx"])
    assert om["pad"] == int(g[name + "_pad"])
    assert om["scale"] == float(g[name + "_scale"])


def test_seed_sequence_key_matches_numpy():
    for seed in (0, 1, 7, 12345, 2 ** 32, 2 ** 32 + 7, 2 ** 64 + 3, 2 ** 130 + 1):
        want = np.random.SeedSequence(seed).generate_state(2, np.uint64)
        assert draws.seed_sequence_key(seed) == tuple(int(x) for x in want)


def test_philox_stream_matches_numpy():
    for seed in (0, 3, 2 ** 33 + 5):
        g = np.random.Generator(np.random.Philox(seed))
        raw = g.bit_generator.random_raw(64)
        got = draws.philox_blocks(draws.seed_sequence_key(seed), 1, 16).reshape(-1)
        np.testing.assert_array_equal(raw, got)


def test_lemire_rejections_match_numpy():
    # a range with a large rejection threshold exercises the rewind path
    for r in (3, 2 ** 31 + 1, 3 * 2 ** 30):
        s = draws.Stream(9)
        g = np.random.Generator(np.random.Philox(9))
        np.testing.assert_array_equal(s.integers(r, 3000), g.integers(0, r, size=3000))
        # the stream stays aligned for the next call
        np.testing.assert_array_equal(s.integers(5, 100), g.integers(0, 5, size=100))


def test_build_sem_hand_properties():
    # tests/test_sketch.py:38-47, 49-53
    row_of, sign = draws.build_sem(5, 40, 1)
    assert row_of.min() >= 0 and row_of.max() < 5
    assert np.all(np.abs(sign) == 1.0)
    row_of, sign = draws.build_sem(2, 100, 7)
    assert math.isclose(np.sqrt(np.sum(sign ** 2)), 10.0)


def test_fast_transform_pad_and_scale():
    # tests/test_sketch.py:123-129
    phase, idx, pad, scale = draws.build_fast_transform(3, 12, 0)
    assert pad == 16 and scale == pytest.approx(np.sqrt(16 / 3))


# --------------------------------------------------------------------------
# kernels (_fast.pyx)


def test_kernels_match_reference(golden):
    g = golden("kernels.npz")
    for name, case in cases.kernel_cases().items():
        kind = case["kind"]
        if kind == "fwht":
            x = np.ascontiguousarray(case["x"].copy())
            O.fwht_rows(x)
            got = x
        elif kind == "gather_dense":
            got = O.sem_gather(case["a"], case["row_of"], case["sign"], case["out_shape"][1])
        elif kind == "scatter_dense":
            got = O.sem_scatter(case["a"], case["row_of"], case["sign"], case["out_shape"][0])
        elif kind == "gather_csc":
            got = O.sem_gather(case["csc"], case["row_of"], case["sign"], case["out_shape"][1])
        else:
            got = O.sem_scatter(case["csc"], case["row_of"], case["sign"], case["out_shape"][0])
        np.testing.assert_array_equal(got, g[name], err_msg=name)


def test_sem_gather_hand_case():
    # tests/test_sketch.py:202-207
    out = O.sem_gather(np.array([[1.0, 2.0, 3.0]]), np.array([0, 0, 1]),
                       np.array([1.0, -1.0, 1.0]), 2)
    np.testing.assert_array_equal(out, [[-1.0, 3.0]])


# --------------------------------------------------------------------------
# factorizations (factor.py)


def test_factor_match_reference(golden):
    g = golden("factor.npz")
    for name, b in cases.factor_cases().items():
        if b.shape[0] >= b.shape[1]:
            p, l, u = O.lu_row_pivot(b)
            np.testing.assert_array_equal(p, g[name + "_row_P"], err_msg=name)
            np.testing.assert_array_equal(l, g[name + "_row_L"], err_msg=name)
            np.testing.assert_array_equal(u, g[name + "_row_U"], err_msg=name)
        bt = b.T if b.shape[0] >= b.shape[1] else b
        q, l, u = O.lu_col_pivot(bt)
        np.testing.assert_array_equal(q, g[name + "_col_Q"], err_msg=name)
        np.testing.assert_array_equal(l, g[name + "_col_L"], err_msg=name)
        np.testing.assert_array_equal(u, g[name + "_col_U"], err_msg=name)


def test_factor_hand_cases():
    # tests/test_factor.py:36-40, 105-109, 160-162
    p, l, u = O.lu_row_pivot(np.array([[0.0, 1.0], [1.0, 0.0]]))
    np.testing.assert_array_equal(p, [1, 0])
    q, l, u = O.lu_col_pivot(np.array([[1.0, 5.0], [0.0, 1.0]]))
    np.testing.assert_array_equal(q, [1, 0])
    np.testing.assert_allclose(l, [[1.0, 0.0], [0.2, 1.0]])
    np.testing.assert_allclose(u, [[5.0, 1.0], [0.0, -0.2]])
    np.testing.assert_allclose(O.left_pseudo_inverse(np.array([[1.0], [1.0]])),
                               [[0.5, 0.5]], atol=1e-15)


def test_pinv_rank_deficient(rng):
    # tests/test_factor.py:194-200
    x = rng(12).standard_normal((20, 3))
    with pytest.raises(O.SingularMatrixError) as exc:
        O.left_pseudo_inverse(np.hstack([x, x[:, :1]]))
    assert exc.value.cond > 1e10


# --------------------------------------------------------------------------
# the whole path (randlu.py:208-276)

PIPES = ["small_dense", "ragged", "sparse", "zero", "lowrank_resample",
         "tall_f32", "sparse_wide", "cfg1"]


@pytest.mark.parametrize("name", PIPES)
def test_pipeline_matches_reference(name, golden):
    g = golden(f"pipe_{name}.npz")
    a, prm = cases.pipeline_cases()[name]
    dense_in = a.toarray() if hasattr(a, "toarray") else a
    assert _sha(np.asarray(dense_in, dtype=np.float64)) == g["a_sha"].item().decode()
    with threadpool_limits(1):
        res = O.sparse_randomized_lu(a, prm, keep=True)
        err = O.approximation_error(a, res)
    assert res["attempt"] == int(g["attempt"])
    # bit-exact: draws, Y, P, L1, both reductions, Q
    for key in ("Y", "P", "red_l", "red_a", "Q"):
        np.testing.assert_array_equal(res[key], g[key], err_msg=key)
    if "L1" in g:
        np.testing.assert_array_equal(res["L1"], g["L1"])
    np.testing.assert_array_equal(res["om2"]["row_of"], g["om2_row_of"])
    np.testing.assert_array_equal(res["om1"]["sample_idx"], g["om1_idx"])
    # same LAPACK/BLAS build single-threaded: L, U identical too
    np.testing.assert_array_equal(res["L"], g["L"])
    np.testing.assert_array_equal(res["U"], g["U"])
    assert err == pytest.approx(float(g["err"]), rel=1e-12, abs=1e-300)


def test_resample_callback_called_twice():
    a, prm = cases.pipeline_cases()["lowrank_resample"]
    calls = []
    O.sparse_randomized_lu(a, prm, on_resample=lambda t, e: calls.append(t))
    assert calls == [0, 1]


# --------------------------------------------------------------------------
# the blocked multithreaded restatement (oracle/lu_blocked.c) used by the
# full-size checks: pinned to the reference's golden factorizations and to
# the numpy restatement above, bit for bit


def test_blocked_lu_matches_reference_goldens(golden):
    g = golden("factor.npz")
    for name, b in cases.factor_cases().items():
        if b.shape[0] >= b.shape[1]:
            p, l, u = O.lu_row_pivot_blocked(b, nthreads=3)
            np.testing.assert_array_equal(p, g[name + "_row_P"], err_msg=name)
            np.testing.assert_array_equal(l, g[name + "_row_L"], err_msg=name)
            np.testing.assert_array_equal(u, g[name + "_row_U"], err_msg=name)
        bt = b.T if b.shape[0] >= b.shape[1] else b
        q, l, u = O.lu_col_pivot_blocked(np.ascontiguousarray(bt.T), nthreads=3)
        np.testing.assert_array_equal(q, g[name + "_col_Q"], err_msg=name)
        np.testing.assert_array_equal(l, g[name + "_col_L"], err_msg=name)
        np.testing.assert_array_equal(u, g[name + "_col_U"], err_msg=name)


@pytest.mark.parametrize("m,k,kind,threads", [
    (2000, 60, "gauss", 4), (5000, 110, "gauss", 7), (3000, 37, "gauss", 1),
    (4000, 40, "lowrank", 3), (600, 40, "ties", 5), (12000, 100, "gauss", 8)])
def test_blocked_lu_matches_numpy_restatement(m, k, kind, threads):
    rng = np.random.default_rng(m + k)
    if kind == "gauss":
        y = rng.standard_normal((m, k))
    elif kind == "lowrank":     # exercises the PIVOT_RTOL branch (factor.py:70-75)
        y = rng.standard_normal((m, 5)) @ rng.standard_normal((5, k))
    else:                       # many exactly tied pivot candidates
        y = rng.integers(-3, 4, (m, k)).astype(np.float64)
    want = O.lu_row_pivot(y)
    got = O.lu_row_pivot_blocked(y, nthreads=threads)
    for w, g_ in zip(want, got):
        np.testing.assert_array_equal(w, g_)
    c = y[: min(k, 64) + 7].T.copy() if kind == "lowrank" else y[:k].T.copy()  # k' x n
    want = O.lu_col_pivot(c)
    got = O.lu_col_pivot_blocked(np.ascontiguousarray(c.T), nthreads=threads)
    for w, g_ in zip(want, got):
        np.testing.assert_array_equal(w, g_)


def test_chunked_sketches_match_restatement():
    import scipy.sparse as sp
    rng = np.random.default_rng(11)
    a = rng.standard_normal((300, 700)).astype(np.float32)
    om = draws.build_composite(40, 160, 700, 3)
    np.testing.assert_array_equal(O.sketch_right_rows(a, om, nthreads=3),
                                  O.apply_sketch_right(O.as_matrix(a.astype(np.float64)), om))
    s = sp.random(300, 700, density=0.02, random_state=1, format="csr")
    np.testing.assert_array_equal(O.sketch_right_rows(s, om),
                                  O.apply_sketch_right(O.as_matrix(s), om))
    om2 = draws.build_composite(30, 120, 300, 4)
    perm = rng.permutation(300)
    for dt in (np.float32, np.float64):
        got = O.sketch_left_cols(a.astype(dt), perm, om2, nthreads=3)
        want = O.apply_sketch_left(om2, a.astype(np.float64)[perm])
        np.testing.assert_array_equal(got, want.T)
