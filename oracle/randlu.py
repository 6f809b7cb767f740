"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement (numpy + the C loops of oracle/kernels.c) of the
reference's sparse randomized LU, used by tests/, by
``__graft_entry__.smoke()`` as the checker and by ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg as the timed CPU port.  The
product path (``paper_1601_04280_b200``) never imports this module.

Every function cites the reference lines it restates; paths are relative
to /root/reference/pkg/src/sparselu/.

Parity pin: tests/test_oracle.py checks this module bit-for-bit against
golden vectors produced by the reference itself (tests/golden/, made by
tests/golden/make_golden.py importing /root/reference in the build
container) and against the reference's own known-answer tests.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time

import numpy as np
from scipy.linalg import solve_triangular
from scipy.sparse import csc_array, issparse

from . import draws

PIVOT_RTOL = 1e-14      # factor.py:19
RANK_RTOL = 1e-10       # factor.py:22
MAX_RESAMPLES = 3       # randlu.py:46

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


class SingularMatrixError(ValueError):
    """errors.py:28-35"""

    def __init__(self, message, cond=float("inf")):
        super().__init__(message)
        self.cond = cond


class DecompositionError(RuntimeError):
    """errors.py:38-39"""


def build() -> str:
    """Compile oracle/kernels.c (gcc) into oracle/_build/liboracle.so."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH)
                < os.path.getmtime(os.path.join(_HERE, "kernels.c"))):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        L.oracle_fwht_rows.argtypes = [P, I, I]
        L.oracle_sem_gather_dense.argtypes = [P, I, I, I, P, P, P, I]
        L.oracle_sem_scatter_dense.argtypes = [P, I, I, I, P, P, P, I]
        L.oracle_sem_gather_csc.argtypes = [P, P, P, I, P, P, P, I]
        L.oracle_sem_scatter_csc.argtypes = [P, P, P, I, P, P, P, I]
        C = ctypes.c_int
        D = ctypes.c_double
        L.oracle_lu_blocked.argtypes = [P, I, I, C, D, P, C, I]
        L.oracle_sketch_right_dense_rows.argtypes = [P, C, I, I, I, P, P, P, I, I, P, I, D, P,
                                                     I, C]
        L.oracle_sketch_right_csr_rows.argtypes = [P, P, P, C, I, P, P, P, I, I, P, I, D, P, I,
                                                   C]
        L.oracle_sketch_left_dense_cols.argtypes = [P, C, I, I, I, P, P, P, P, I, I, P, I, D, P,
                                                    I, C]
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


# --------------------------------------------------------------------------
# input coercion: matrix.py:54-77 (dense -> F-order float64 copy; sparse ->
# CSC int64, duplicates summed, sorted indices)


def as_matrix(a):
    if issparse(a):
        c = csc_array(a, copy=True).astype(np.float64)
        c.sum_duplicates()
        c.sort_indices()
        c.indices = np.ascontiguousarray(c.indices, dtype=np.int64)
        c.indptr = np.ascontiguousarray(c.indptr, dtype=np.int64)
        return c
    return np.array(a, dtype=np.float64, order="F")


# --------------------------------------------------------------------------
# kernels (C restatement, oracle/kernels.c)


def fwht_rows(x):
    """_kernels fwht_rows (_fast.pyx:23-41): in place, C-contiguous."""
    assert x.flags.c_contiguous and x.dtype == np.float64
    lib().oracle_fwht_rows(_p(x), x.shape[0], x.shape[1])


def sem_gather(a, row_of, sign, l):
    """apply_sem_adjoint_right (sketch.py:285-301): a @ S^T, m x l F-order."""
    row_of = np.ascontiguousarray(row_of, dtype=np.int64)
    sign = np.ascontiguousarray(sign, dtype=np.float64)
    if issparse(a):
        out = np.zeros((a.shape[0], l), order="F")
        lib().oracle_sem_gather_csc(_p(a.data), _p(a.indices), _p(a.indptr),
                                    a.shape[1], _p(row_of), _p(sign), _p(out),
                                    out.shape[0])
        return out
    a = np.asfortranarray(a, dtype=np.float64)
    out = np.zeros((a.shape[0], l), order="F")
    lib().oracle_sem_gather_dense(_p(a), a.shape[0], a.shape[1], a.shape[0],
                                  _p(row_of), _p(sign), _p(out), out.shape[0])
    return out


def sem_scatter(a, row_of, sign, l):
    """_sem_mul_left (sketch.py:304-313): S @ a, l x cols F-order."""
    row_of = np.ascontiguousarray(row_of, dtype=np.int64)
    sign = np.ascontiguousarray(sign, dtype=np.float64)
    if issparse(a):
        out = np.zeros((l, a.shape[1]), order="F")
        lib().oracle_sem_scatter_csc(_p(a.data), _p(a.indices), _p(a.indptr),
                                     a.shape[1], _p(row_of), _p(sign), _p(out),
                                     out.shape[0])
        return out
    a = np.asfortranarray(a, dtype=np.float64)
    out = np.zeros((l, a.shape[1]), order="F")
    lib().oracle_sem_scatter_dense(_p(a), a.shape[0], a.shape[1], a.shape[0],
                                   _p(row_of), _p(sign), _p(out), out.shape[0])
    return out


def fast_adjoint_right(b, om):
    """_fast_adjoint_right, hadamard lane (sketch.py:322-335)."""
    m = b.shape[0]
    pad, l = om["pad"], om["l"]
    x = np.zeros((m, pad))
    x[:, :l] = b * om["phase"]
    fwht_rows(x)
    mult = om["scale"] / math.sqrt(pad)
    return x[:, om["sample_idx"]] * mult


def fast_mul_left(mm, om):
    """_fast_mul_left, hadamard lane (sketch.py:338-349)."""
    c = mm.shape[1]
    pad, l = om["pad"], om["l"]
    x = np.zeros((c, pad))
    x[:, :l] = mm.T * om["phase"]
    fwht_rows(x)
    return np.asfortranarray((x[:, om["sample_idx"]] * (om["scale"] / math.sqrt(pad))).T)


def apply_sketch_right(a, om):
    """sketch.py:362-368"""
    return fast_adjoint_right(sem_gather(a, om["row_of"], om["sign"], om["l"]), om)


def apply_sketch_left(om, a):
    """sketch.py:371-378"""
    return fast_mul_left(sem_scatter(a, om["row_of"], om["sign"], om["l"]), om)


# --------------------------------------------------------------------------
# factorizations: factor.py


def lu_row_pivot(b):
    """factor.py:49-77.  Returns (perm, L lower-trapezoidal, U)."""
    m, k = b.shape
    if m < k:
        raise ValueError(f"need rows >= cols, got {m} x {k}")
    w = np.array(b, order="F", dtype=np.float64)
    perm = np.arange(m)
    thresh = PIVOT_RTOL * np.linalg.norm(w)
    for i in range(k):
        p = i + int(np.argmax(np.abs(w[i:, i])))
        if p != i:
            w[[i, p], :] = w[[p, i], :]
            perm[[i, p]] = perm[[p, i]]
        piv = w[i, i]
        if abs(piv) > thresh:
            w[i + 1:, i] /= piv
            w[i + 1:, i + 1:] -= np.outer(w[i + 1:, i], w[i, i + 1:])
        else:
            w[i + 1:, i] = 0.0
    lower = np.tril(w[:, :k], -1)
    lower[np.arange(k), np.arange(k)] = 1.0
    # Matrix._owned stores F-order (matrix.py:93-104); BLAS sees that layout
    return perm, np.asfortranarray(lower), np.asfortranarray(np.triu(w[:k, :k]))


def lu_col_pivot(mat):
    """factor.py:80-109.  Returns (q, L unit lower k x k, U k x n)."""
    k, n = mat.shape
    if k > n:
        raise ValueError(f"need rows <= cols, got {k} x {n}")
    w = np.array(mat, order="F", dtype=np.float64)
    q = np.arange(n)
    thresh = PIVOT_RTOL * np.linalg.norm(w)
    for i in range(k):
        p = i + int(np.argmax(np.abs(w[i, i:])))
        if p != i:
            w[:, [i, p]] = w[:, [p, i]]
            q[[i, p]] = q[[p, i]]
        piv = w[i, i]
        if abs(piv) > thresh:
            w[i + 1:, i] /= piv
            w[i + 1:, i + 1:] -= np.outer(w[i + 1:, i], w[i, i + 1:])
        else:
            w[i + 1:, i] = 0.0
    lower = np.tril(w[:, :k], -1)
    lower[np.arange(k), np.arange(k)] = 1.0
    return q, np.asfortranarray(lower), np.asfortranarray(np.triu(w))


def _lu_blocked(w, mode, thresh, nthreads):
    w = np.array(w, dtype=np.float64, order="C")          # a copy: factorized in place
    M, k = w.shape
    perm = np.empty(M, dtype=np.int64)
    lib().oracle_lu_blocked(_p(w), M, k, mode, float(thresh), _p(perm), int(nthreads), 32)
    return w, perm


def lu_row_pivot_blocked(y, nthreads=0, thresh=None):
    """lu_row_pivot (factor.py:49-77) by the blocked multithreaded C
    restatement (oracle/lu_blocked.c), bit-identical to lu_row_pivot; for
    the full-size checks.  ``thresh`` defaults to PIVOT_RTOL·||Y||_F computed
    like the reference (norm of the F-order working copy).  Returns (perm,
    L m x k C-order, U k x k)."""
    m, k = y.shape
    if m < k:
        raise ValueError(f"need rows >= cols, got {m} x {k}")
    if thresh is None:
        thresh = PIVOT_RTOL * np.linalg.norm(np.asfortranarray(y, dtype=np.float64))
    w, perm = _lu_blocked(y, 0, thresh, nthreads)
    u = np.triu(w[:k, :k])
    w[:k, :k] = np.tril(w[:k, :k], -1)
    w[np.arange(k), np.arange(k)] = 1.0
    return perm, w, u


def lu_col_pivot_blocked(core_t, nthreads=0, thresh=None):
    """lu_col_pivot (factor.py:80-109) of core = core_t^T by the blocked C
    restatement, on core_t (n x k: rows of core_t are columns of core).
    Returns (q, L~ k x k, U k x n)."""
    n, k = core_t.shape
    if k > n:
        raise ValueError(f"need rows <= cols, got {k} x {n}")
    if thresh is None:
        thresh = PIVOT_RTOL * np.linalg.norm(np.asfortranarray(np.asarray(core_t).T))
    w, q = _lu_blocked(core_t, 1, thresh, nthreads)
    lower = np.triu(w[:k, :k], 1).T.copy()
    lower[np.arange(k), np.arange(k)] = 1.0
    return q, lower, np.triu(w.T)


def sketch_right_rows(a_rows, om, nthreads=0):
    """apply_sketch_right (sketch.py:362-368) of a block of rows of A (C
    order fp32/fp64, or a scipy CSR block with ascending indices), multi-
    threaded C (oracle/lu_blocked.c); bit-identical to apply_sketch_right
    on the same rows.  Returns rows x k (C order)."""
    row_of = np.ascontiguousarray(om["row_of"], dtype=np.int64)
    sign = np.ascontiguousarray(om["sign"], dtype=np.float64)
    phase = np.ascontiguousarray(om["phase"], dtype=np.float64)
    sample = np.ascontiguousarray(om["sample_idx"], dtype=np.int64)
    k, l, pad = len(sample), om["l"], om["pad"]
    mult = om["scale"] / math.sqrt(pad)
    rows = a_rows.shape[0]
    y = np.empty((rows, k))
    if issparse(a_rows):
        indptr = np.ascontiguousarray(a_rows.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(a_rows.indices, dtype=np.int32)
        vals = np.ascontiguousarray(a_rows.data)
        dt = 0 if vals.dtype == np.float32 else 1
        vals = vals if dt == 0 else vals.astype(np.float64)
        lib().oracle_sketch_right_csr_rows(_p(indptr), _p(indices), _p(vals), dt, rows,
                                           _p(row_of), _p(sign), _p(phase), l, pad, _p(sample),
                                           k, mult, _p(y), k, int(nthreads))
        return y
    a_rows = np.ascontiguousarray(a_rows)
    dt = 0 if a_rows.dtype == np.float32 else 1
    if dt:
        a_rows = a_rows.astype(np.float64, copy=False)
    lib().oracle_sketch_right_dense_rows(_p(a_rows), dt, rows, a_rows.shape[1], a_rows.shape[1],
                                         _p(row_of), _p(sign), _p(phase), l, pad, _p(sample), k,
                                         mult, _p(y), k, int(nthreads))
    return y


def sketch_left_cols(a_cols, perm, om, nthreads=0):
    """apply_sketch_left (sketch.py:371-378) of P·A restricted to a block of
    columns: ``a_cols`` is the m x nb block of A (C order fp32/fp64, rows in
    A's order), ``perm`` P's indices.  Returns nb x k2 = the block's columns
    of (Omega2 P A)^T, bit-identical to apply_sketch_left(om, A[perm])."""
    a_cols = np.ascontiguousarray(a_cols)
    dt = 0 if a_cols.dtype == np.float32 else 1
    if dt:
        a_cols = a_cols.astype(np.float64, copy=False)
    m, nb = a_cols.shape
    perm = np.ascontiguousarray(perm, dtype=np.int64)
    row_of = np.ascontiguousarray(om["row_of"], dtype=np.int64)
    sign = np.ascontiguousarray(om["sign"], dtype=np.float64)
    phase = np.ascontiguousarray(om["phase"], dtype=np.float64)
    sample = np.ascontiguousarray(om["sample_idx"], dtype=np.int64)
    k, l, pad = len(sample), om["l"], om["pad"]
    out = np.empty((nb, k))
    lib().oracle_sketch_left_dense_cols(_p(a_cols), dt, m, nb, nb, _p(perm), _p(row_of),
                                        _p(sign), _p(phase), l, pad, _p(sample), k,
                                        om["scale"] / math.sqrt(pad), _p(out), k, int(nthreads))
    return out


def left_pseudo_inverse(mat):
    """factor.py:112-130 (Householder QR, sigma-ratio rank check)."""
    p, q = mat.shape
    if p < q:
        raise ValueError(f"need rows >= cols, got {p} x {q}")
    qf, rf = np.linalg.qr(mat, mode="reduced")
    sv = np.linalg.svd(rf, compute_uv=False)
    if sv[0] == 0.0 or sv[-1] <= RANK_RTOL * sv[0]:
        cond = float("inf") if sv[-1] == 0.0 else float(sv[0] / sv[-1])
        raise SingularMatrixError(
            f"matrix is numerically rank deficient (condition estimate {cond:.3e})",
            cond=cond)
    return np.asfortranarray(solve_triangular(rf, qf.conj().T))


def matmul(a, b):
    """matrix.py:219-230 on F-order operands (Matrix._owned layout)."""
    return np.asfortranarray(np.asfortranarray(a) @ np.asfortranarray(b))


def permute_rows(perm, a):
    """matrix.py:201-207"""
    if issparse(a):
        return as_matrix(a[perm, :])
    return np.asfortranarray(a[perm, :])


# --------------------------------------------------------------------------
# the pipeline: randlu.py:208-276


def _attempt(a, params, attempt, keep):
    m, n = a.shape
    el = {}
    tic = time.perf_counter()
    s1 = params["seed"] + 2 * attempt
    s2 = params["seed"] + 2 * attempt + 1
    om1 = draws.build_composite(params["k1"], params["l1"], n, s1)
    om2 = draws.build_composite(params["k2"], params["l2"], m, s2)
    y = apply_sketch_right(a, om1)
    el["sketch1"] = time.perf_counter() - tic

    tic = time.perf_counter()
    perm, l1, _ = lu_row_pivot(y)
    el["lu1"] = time.perf_counter() - tic

    tic = time.perf_counter()
    red_l = apply_sketch_left(om2, l1)
    pa = permute_rows(perm, a)
    red_a = apply_sketch_left(om2, pa)
    del pa
    el["sketch2"] = time.perf_counter() - tic

    tic = time.perf_counter()
    pinv = left_pseudo_inverse(red_l)
    core = matmul(pinv, red_a)
    el["pinv"] = time.perf_counter() - tic

    tic = time.perf_counter()
    q, lt, u = lu_col_pivot(core)
    lfinal = matmul(l1, lt)
    el["lu2"] = time.perf_counter() - tic
    res = dict(P=perm, Q=q, L=lfinal, U=u, elapsed=el, attempt=attempt)
    if keep:
        res.update(Y=y, L1=l1, red_l=red_l, red_a=red_a, pinv=pinv, core=core,
                   Lt=lt, om1=om1, om2=om2)
    return res


def check_params(params, m, n):
    """randlu.py:69-95"""
    r, k1, l1, k2, l2 = (params[x] for x in ("r", "k1", "l1", "k2", "l2"))
    if r < 1 or not r <= k1 <= k2 or not k1 < l1 or not k2 < l2:
        raise ValueError("invalid RandLuParams invariants")
    if l1 > n or l2 > m or k2 > m or k1 > m:
        raise ValueError("params do not fit the matrix")


def sparse_randomized_lu(a, params, keep=False, on_resample=None):
    """randlu.py:208-243.  ``params``: dict with r, k1, l1, k2, l2, seed.
    ``a``: dense ndarray or scipy sparse.  Returns a dict with P, Q, L, U,
    elapsed (+ intermediates when keep=True)."""
    a = as_matrix(a)
    m, n = a.shape
    check_params(params, m, n)
    t0 = time.perf_counter()
    last = None
    for attempt in range(1 + MAX_RESAMPLES):
        try:
            res = _attempt(a, params, attempt, keep)
            res["elapsed"]["total"] = time.perf_counter() - t0
            return res
        except SingularMatrixError as err:
            last = err
            if on_resample is not None:
                on_resample(attempt, err)
    raise DecompositionError("reduced system stayed rank deficient") from last


def approximation_error(a, res, block_cols=256):
    """randlu.py:279-302: ||L U - P A Q||_F in column blocks."""
    a = as_matrix(a)
    m, n = a.shape
    perm, cols = np.asarray(res["P"]), np.asarray(res["Q"])
    ld, ud = np.asarray(res["L"]), np.asarray(res["U"])
    acc = 0.0
    for start in range(0, n, block_cols):
        sel = cols[start:start + block_cols]
        prod = ld @ ud[:, start:start + block_cols]
        if issparse(a):
            block = a[:, sel].toarray()[perm, :]
        else:
            block = a[np.ix_(perm, sel)]
        acc += float(np.sum(np.abs(prod - block) ** 2))
    return math.sqrt(acc)


def _qr_longdouble(mat):
    """Householder QR in x87 extended precision (64-bit mantissa)."""
    R = np.array(mat, dtype=np.longdouble)
    p, q = R.shape
    Q = np.eye(p, dtype=np.longdouble)
    for j in range(q):
        x = R[j:, j]
        nx = np.sqrt(np.sum(x * x))
        if nx == 0:
            continue
        v = x.copy()
        v[0] += nx if x[0] >= 0 else -nx
        v /= np.sqrt(np.sum(v * v))
        R[j:, j:] -= 2 * np.outer(v, v @ R[j:, j:])
        Q[:, j:] -= 2 * np.outer(Q[:, j:] @ v, v)
    return Q[:, :q], R[:q, :q]


def forward_error_band(red_l, red_a, l1):
    """How far the reference's own L, U sit from the (nearly) exact answer.

    Re-runs the tail of the pipeline (pinv, core = pinv·red_a, lu_col_pivot,
    L = L1·L~) with pinv and core formed in extended precision, from the
    reference's bit-exact intermediates.  The distance between these factors
    and the reference's is the reference's own forward error; any other
    correct fp64 implementation (a different but equally stable QR/GEMM)
    lands at a comparable distance.  Returns (q, L, U)."""
    qf, rf = _qr_longdouble(red_l)
    k = rf.shape[0]
    b = qf.T.copy()
    x = np.zeros_like(b)
    for i in range(k - 1, -1, -1):
        x[i] = (b[i] - rf[i, i + 1:] @ x[i + 1:]) / rf[i, i]
    core = (x @ np.asarray(red_a, dtype=np.longdouble)).astype(np.float64)
    q, lt, u = lu_col_pivot_blocked(np.ascontiguousarray(core.T))
    return q, matmul(l1, lt), u


def default_params(r, m, n, seed=0):
    """randlu.py:117-143 (practical mode)."""
    if not 1 <= r <= min(m, n) / 2:
        raise ValueError("need 1 <= r <= min(m,n)/2")
    k1 = min(n - 1, r + 8)
    k2 = min(m - 1, k1 + 8)
    l1 = min(n, 4 * k1)
    l2 = min(m, 4 * k2)
    return dict(r=r, k1=k1, l1=l1, k2=k2, l2=l2, seed=seed)
