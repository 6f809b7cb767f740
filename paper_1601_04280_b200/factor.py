"""Pivoted LUs and the left pseudo-inverse on the device (factor.py).

``lu_row_pivot`` / ``lu_col_pivot`` run the persistent CUDA kernel K2/K5
(bit-exact replays of factor.py:49-77 / :80-109).  ``left_pseudo_inverse``
keeps the reference's Householder-QR formulation and sigma-ratio rank test
(factor.py:112-130) in libsrlu kernels; ``dgemm`` is libsrlu's FP64
tensor-core (DMMA) GEMM.
"""

from __future__ import annotations

import torch

from . import _lib
from .errors import ShapeError, SingularMatrixError
from .matrix import Matrix, Permutation

PIVOT_RTOL = 1e-14   # factor.py:19 (compiled into lu.cu)
RANK_RTOL = 1e-10    # factor.py:22


class PivotedLU:
    """P B = L U, unit lower-trapezoidal L, square upper U (factor.py:25-34)."""

    __slots__ = ("P", "L", "U")

    def __init__(self, P, L, U):
        self.P, self.L, self.U = P, L, U


class ColPivotedLU:
    """M Q = L U, unit lower L, upper-trapezoidal U (factor.py:37-46)."""

    __slots__ = ("Q", "L", "U")

    def __init__(self, Q, L, U):
        self.Q, self.L, self.U = Q, L, U


def lu_row_pivot_dev(y: torch.Tensor, want_u: bool = False, stream=None):
    """K2 on a row-major fp64 m x k device tensor (overwritten).
    Returns (perm int64[m] device, L m x k, U k x k or None)."""
    L = _lib.lib()
    m, k = y.shape
    if m < k:
        raise ShapeError(f"need rows >= cols, got {m} x {k}")
    dev = y.device
    perm = torch.empty(m, dtype=torch.int64, device=dev)
    lo = torch.empty(m, k, dtype=torch.float64, device=dev)
    up = torch.zeros(k, k, dtype=torch.float64, device=dev) if want_u else None
    ws = _lib.workspace(L.srlu_lu_workspace(m, k), dev)
    _lib.check(L.srlu_lu_rowpiv(_lib.ptr(y), m, k, y.stride(0), _lib.ptr(perm), _lib.ptr(lo),
                                lo.stride(0), _lib.ptr(up), k, 0, _lib.ptr(ws), ws.numel(),
                                _lib.stream_handle(stream)), "lu_row_pivot")
    return perm, lo, up


def lu_col_pivot_dev(ct: torch.Tensor, stream=None, reserve_sms=0):
    """K5 on core^T (n x k row-major fp64 device tensor, overwritten).
    Returns (q int64[n], Lt k x k, UT n x k) with U = UT^T.  ``reserve_sms``
    SMs stay out of the cooperative grid (a side-stream kernel runs there)."""
    L = _lib.lib()
    n, k = ct.shape
    if k > n:
        raise ShapeError(f"need rows <= cols, got {k} x {n}")
    dev = ct.device
    q = torch.empty(n, dtype=torch.int64, device=dev)
    lt = torch.zeros(k, k, dtype=torch.float64, device=dev)
    ut = torch.empty(n, k, dtype=torch.float64, device=dev)
    ws = _lib.workspace(L.srlu_lu_workspace(n, k), dev)
    _lib.check(L.srlu_lu_colpiv(_lib.ptr(ct), n, k, ct.stride(0), _lib.ptr(q), _lib.ptr(lt),
                                lt.stride(0), _lib.ptr(ut), ut.stride(0), reserve_sms, _lib.ptr(ws),
                                ws.numel(), _lib.stream_handle(stream)), "lu_col_pivot")
    return q, lt, ut


def _dense_f64(b) -> torch.Tensor:
    if isinstance(b, Matrix):
        t = b.to_dense()
    elif isinstance(b, torch.Tensor):
        t = b
    else:
        t = Matrix(b).to_dense()
    if not t.is_cuda:
        t = t.cuda()
    return t.to(torch.float64).contiguous().clone()


def lu_row_pivot(b) -> PivotedLU:
    """factor.py:49-77 on the device."""
    y = _dense_f64(b)
    if y.shape[0] < y.shape[1]:
        raise ShapeError(f"need rows >= cols, got {y.shape[0]} x {y.shape[1]}")
    perm, lo, up = lu_row_pivot_dev(y, want_u=True)
    return PivotedLU(Permutation(perm.cpu().numpy(), perm), Matrix.from_device(lo),
                     Matrix.from_device(up))


def lu_col_pivot(mat) -> ColPivotedLU:
    """factor.py:80-109 on the device."""
    c = _dense_f64(mat)
    k, n = c.shape
    if k > n:
        raise ShapeError(f"need rows <= cols, got {k} x {n}")
    q, lt, ut = lu_col_pivot_dev(c.t().contiguous())
    return ColPivotedLU(Permutation(q.cpu().numpy(), q), Matrix.from_device(lt),
                        Matrix.from_device(ut.t().contiguous()))


class RankTest:
    """Device state of one rank test (factor.py:122-128): the certified
    stats[8] of srlu_qr_rank_certified and the QR workspace (R) for the
    exact fallback."""

    __slots__ = ("stats", "ws", "k1", "k2")

    def __init__(self, stats, ws, k1, k2):
        self.stats, self.ws, self.k1, self.k2 = stats, ws, k1, k2

    def record_stream(self, stream):
        self.stats.record_stream(stream)
        self.ws.record_stream(stream)


def pinv_dev(m_t: torch.Tensor, stream=None, rank_event=False):
    """pinv of M = m_t^T (k2 x k1) on the device (factor.py:112-130).
    ``m_t``: k1 x k2 row-major fp64.  Returns (pinvT k2 x k1, RankTest[,
    event]).  The rank test is enqueued AFTER the pinv (same stream) so a
    consumer of pinvT can wait on the returned event and overlap the rank
    test; the caller decides singularity after its one host sync
    (``check_rank``).  libsrlu's Householder QR runs in one CTA when M fits
    its shared memory, else on one thread-block cluster (k1 <= 576)."""
    L = _lib.lib()
    m_t = m_t.contiguous()
    k1, k2 = m_t.shape
    if k2 < k1:
        raise ShapeError(f"need rows >= cols, got {k2} x {k1}")
    dev = m_t.device
    stats = torch.empty(8, dtype=torch.float64, device=dev)
    sh = _lib.stream_handle(stream)
    ev = torch.cuda.Event()
    pinv_t = torch.empty(k2, k1, dtype=torch.float64, device=dev)
    ws = _lib.workspace(L.srlu_qr_pinv_workspace(k1, k2), dev)
    _lib.check(L.srlu_qr_pinv(_lib.ptr(m_t), k1, k2, m_t.stride(0), _lib.ptr(pinv_t),
                              pinv_t.stride(0), _lib.ptr(stats), _lib.ptr(ws), ws.numel(), sh),
               "qr_pinv")
    ev.record(stream)
    _lib.check(L.srlu_qr_rank_certified(_lib.ptr(ws), k1, k2, _lib.ptr(pinv_t), pinv_t.stride(0),
                                        _lib.ptr(stats), sh), "qr_rank")
    rt = RankTest(stats, ws, k1, k2)
    if rank_event:
        return pinv_t, rt, ev
    return pinv_t, rt


def dgemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None, stream=None,
          b_lower: bool = False):
    """out = a @ b (row-major fp64) on the FP64 tensor cores (libsrlu
    srlu_dgemm_ex, DMMA): core = pinv . (Omega2 P A) (randlu.py:267) and
    L = L1 . L~ (randlu.py:272).  ``b_lower``: b is lower triangular (L~);
    its zero blocks are skipped."""
    L = _lib.lib()
    a = a if a.stride(1) == 1 else a.contiguous()
    b = b if b.stride(1) == 1 else b.contiguous()
    M, K = a.shape
    K2, N = b.shape
    if K != K2:
        raise ShapeError(f"inner dimensions differ: {tuple(a.shape)} x {tuple(b.shape)}")
    if a.dtype != torch.float64 or b.dtype != torch.float64:
        raise ShapeError("dgemm needs float64 operands")
    if out is None:
        out = torch.empty(M, N, dtype=torch.float64, device=a.device)
    _lib.check(L.srlu_dgemm_ex(_lib.ptr(a), a.stride(0), _lib.ptr(b), b.stride(0), _lib.ptr(out),
                               out.stride(0), M, N, K, 1 if b_lower else 0,
                               _lib.stream_handle(stream)), "dgemm")
    return out


def check_rank(stats_host, rank: RankTest | None = None, stream=None):
    """factor.py:123-128 on the certified bounds of srlu_qr_rank_certified;
    undecided (flag 2: the bounds straddle 1e-10) -> the singular values of
    R themselves (srlu_rank_exact, one-sided Jacobi on the device), like the
    reference.  Returns the stats the decision was made on."""
    st = [float(x) for x in stats_host]
    if st[3] == 2.0:
        if rank is None:
            raise RuntimeError("undecided rank test needs the device R")
        L = _lib.lib()
        dev = rank.ws.device
        ex = torch.empty(4, dtype=torch.float64, device=dev)
        ws = _lib.workspace(L.srlu_rank_exact_workspace(rank.k1), dev)
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        _lib.check(L.srlu_rank_exact(_lib.ptr(rank.ws), rank.k1, rank.k2, _lib.ptr(ws),
                                     ws.numel(), _lib.ptr(ex), _lib.stream_handle(s)),
                   "rank_exact")
        st = [float(x) for x in ex.cpu()] + [0.0] * 4
        st[7] = 1.0   # decided on the exact singular values
    smax, smin, cond, singular = st[:4]
    if singular:
        cond = float("inf") if smin == 0.0 else float(smax / smin)
        raise SingularMatrixError(
            f"matrix is numerically rank deficient (condition estimate {cond:.3e})", cond=cond)
    return st


def left_pseudo_inverse(mat) -> Matrix:
    """factor.py:112-130 on the device."""
    m = _dense_f64(mat)
    p, q = m.shape
    if p < q:
        raise ShapeError(f"need rows >= cols, got {p} x {q}")
    pinv_t, rt = pinv_dev(m.t().contiguous())
    check_rank(rt.stats.cpu().numpy(), rt)
    return Matrix.from_device(pinv_t.t().contiguous())
