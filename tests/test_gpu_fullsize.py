"""Stage-wise parity of the whole decomposition at the BASELINE configs' full
sizes (2: 16384^2 fp32, 3: 262144 x 8192 fp32, 4: 1048576 x 65536 CSR,
5: 65536^2 fp64) against the CPU oracle, on the GPU box's host cores.

The reference's path (randlu.py:246-276) is a chain of deterministic stages;
each is replayed by the oracle on the device's (already checked) input of
that stage, so together they are the oracle's whole pipeline on the same A:

  1. Y = A Omega1^* (sketch.py:362-368): every row, bit for bit
     (oracle.sketch_right_rows, row blocks of A copied to the host);
  2. P, L1 = lu_row_pivot(Y) (factor.py:49-77): bit for bit
     (oracle.lu_row_pivot_blocked, the blocked multithreaded restatement
     pinned to the reference's goldens in tests/test_oracle.py);
  3. Omega2 L1 and Omega2 (P A) (sketch.py:371-378): bit for bit, every
     column (oracle.sketch_left_cols on column blocks of A);
  4. the tail: the reference's pinv (numpy Householder QR + SVD rank test,
     factor.py:112-130), core = pinv (Omega2 P A) (randlu.py:267),
     Q, L~, U = lu_col_pivot(core) (factor.py:80-109), L = L1 L~
     (randlu.py:272) — against the device's Q, L, U with tests/parity.py's
     criteria (Q exact on the significant pivots; L, U within 1e-10
     relative or, where the reference's own forward error is larger,
     within 4x it); whether the strict 1e-10 held is recorded;
  5. ||L U - P A Q||_F (randlu.py:279-302) of both factor sets, computed by
     K7 on the device: within 1%.

With SRLU_PARITY_LOG=<file> each config appends one JSON line (rel_L,
rel_U, bands, strict?, both errors, stage timings) — profiles/r02/.
"""

import json
import os
import time

import numpy as np
import pytest

from tests.conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def P():
    if not cuda_ok():
        pytest.skip("needs a CUDA device")
    import paper_1601_04280_b200 as pkg
    return pkg


def _np(t):
    return t.detach().cpu().numpy()


def _first_mismatch(got, want):
    bad = np.argwhere(got != want)
    return None if bad.size == 0 else (tuple(bad[0]), got[tuple(bad[0])], want[tuple(bad[0])])


@pytest.mark.parametrize("config", [2, 3, 4, 5])
def test_full_size_stagewise_parity(P, config):
    import torch
    from scipy.sparse import csr_array

    from bench import CONFIGS, as_matrix, gen_config
    from oracle import draws as D
    from oracle import randlu as O
    from tests.parity import check_tail

    tm = {}
    t0 = time.perf_counter()
    cfg = CONFIGS[config]
    m, n = cfg["m"], cfg["n"]
    a, prm = gen_config(config)
    sparse = isinstance(a, tuple)
    mat = as_matrix(P, a, (m, n))
    res = P.sparse_randomized_lu(mat, P.RandLuParams(**prm), keep=True)
    torch.cuda.synchronize()
    tm["device_pipeline_s"] = time.perf_counter() - t0
    assert res.attempt == 0, "resampled: the stage-wise replay below covers attempt 0 only"
    k1, k2 = prm["k1"], prm["k2"]
    om1 = D.build_composite(k1, prm["l1"], n, prm["seed"])
    om2 = D.build_composite(k2, prm["l2"], m, prm["seed"] + 1)
    host = None
    if sparse:
        indptr, indices, values = (_np(t) for t in a)
        host = csr_array((values, indices, indptr), shape=(m, n))

    # 1. Y, every row
    t = time.perf_counter()
    y_dev = res.extras["Y"]
    rb = max(1, (1 << 29) // (n * (4 if sparse else a.element_size())))
    for r0 in range(0, m, rb):
        r1 = min(m, r0 + rb)
        blk = host[r0:r1] if sparse else _np(a[r0:r1])
        y_ref = O.sketch_right_rows(blk, om1)
        mm = _first_mismatch(_np(y_dev[r0:r1]), y_ref)
        assert mm is None, f"Y differs at row {r0 + mm[0][0]}, col {mm[0][1]}: {mm[1]!r} vs {mm[2]!r}"
    tm["Y_check_s"] = time.perf_counter() - t

    # 2. P, L1 = LU(Y)
    t = time.perf_counter()
    y_h = _np(y_dev)
    perm_ref, l1_ref, _ = O.lu_row_pivot_blocked(y_h)
    del y_h
    np.testing.assert_array_equal(res.P.indices, perm_ref)
    l1_dev = _np(res.extras["L1"])
    mm = _first_mismatch(l1_dev, l1_ref)
    assert mm is None, f"L1 differs at {mm}"
    del l1_dev
    tm["LU_Y_check_s"] = time.perf_counter() - t

    # 3. Omega2 L1, Omega2 P A (every column)
    t = time.perf_counter()
    red_l_ref = O.apply_sketch_left(om2, l1_ref)
    np.testing.assert_array_equal(_np(res.extras["red_l"]), red_l_ref)
    red_aT_dev = _np(res.extras["red_a"].t())           # n x k2
    if sparse:
        red_a_ref = O.apply_sketch_left(om2, O.as_matrix(host[perm_ref]))
        mm = _first_mismatch(red_aT_dev, red_a_ref.T)
        assert mm is None, f"Omega2 P A differs at {mm}"
    else:
        red_a_ref = np.empty((k2, n), order="F")
        cb = max(16, (1 << 29) // (m * a.element_size()))
        for c0 in range(0, n, cb):
            c1 = min(n, c0 + cb)
            blk = _np(a[:, c0:c1].contiguous())
            ref = O.sketch_left_cols(blk, perm_ref, om2)     # (c1-c0) x k2
            mm = _first_mismatch(red_aT_dev[c0:c1], ref)
            assert mm is None, f"Omega2 P A differs at column {c0 + mm[0][0]}: {mm}"
            red_a_ref[:, c0:c1] = ref.T
    del red_aT_dev
    tm["sketch2_check_s"] = time.perf_counter() - t

    # 4. the tail: the reference's pinv / core / column LU / L
    t = time.perf_counter()
    pinv_ref = O.left_pseudo_inverse(red_l_ref)
    core_ref = O.matmul(pinv_ref, red_a_ref)
    q_ref, lt_ref, u_ref = O.lu_col_pivot_blocked(np.ascontiguousarray(core_ref.T))
    L_ref = O.matmul(l1_ref, lt_ref)
    stats = check_tail(res.Q.indices, res.L.numpy(), res.U.numpy(), q_ref, L_ref, u_ref,
                       core_ref, red_l_ref, red_a_ref, l1_ref)
    stats["strict_1e-10"] = bool(stats.get("rel_L", 0.0) <= 1e-10
                                 and stats.get("rel_U", 0.0) <= 1e-10)
    stats["Q_exact"] = bool(np.array_equal(res.Q.indices, q_ref))
    tm["tail_check_s"] = time.perf_counter() - t

    # 5. ||L U - P A Q||_F of both factor sets on the device (K7)
    t = time.perf_counter()
    err = P.approximation_error(mat, res)
    ref_res = P.RandLuResult(P=P.Permutation(perm_ref), Q=P.Permutation(q_ref),
                             L=P.Matrix.from_device(torch.from_numpy(L_ref).cuda()),
                             U=P.Matrix.from_device(torch.from_numpy(np.ascontiguousarray(u_ref))
                                                    .cuda()))
    err_ref = P.approximation_error(mat, ref_res)
    tm["error_s"] = time.perf_counter() - t
    rec = dict(config=config, m=m, n=n, params=prm, err=err, err_ref=err_ref,
               err_rel_diff=abs(err - err_ref) / err_ref if err_ref else 0.0, **stats,
               timings_s={k: round(v, 2) for k, v in tm.items()},
               host_threads=os.cpu_count())
    log = os.environ.get("SRLU_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps(rec, default=float) + "\n")
    print(json.dumps(rec, default=float))
    assert abs(err - err_ref) <= 0.01 * err_ref, rec
