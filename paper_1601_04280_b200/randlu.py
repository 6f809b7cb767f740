"""Randomized low-rank pivoted LU on B200 — the drop-in for the reference's
``sparse_randomized_lu`` (randlu.py:208-276).

Same signature, parameter dataclass, result dataclass, error types,
resample semantics (attempt t draws from sub-seeds seed+2t / seed+2t+1,
up to MAX_RESAMPLES retries, warnings on the module logger) and the same
``elapsed`` keys; every stage runs on the GPU:

  sketch1  K0 draws + K1 fused CountSketch/FWHT stream over A  -> Y
  lu1      K2 persistent row-pivoted LU of Y                   -> P, L1
  sketch2  K3 fused left sketch of L1 and of P·A (P·A never materialised)
  pinv     Householder QR + rank test + core = pinv · (Omega2 P A)
  lu2      K5 persistent column-pivoted LU of core; L = L1 · L~

Stage times come from CUDA events on the launching stream; the host
synchronises once per attempt (rank test + non-finite flag).
"""

from __future__ import annotations

import logging
import os
import math
import threading
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from .errors import DecompositionError, ParameterError, ShapeError, SingularMatrixError
from .factor import check_rank, dgemm, lu_col_pivot_dev, lu_row_pivot_dev, pinv_dev
from .matrix import COMPLEX, REAL, Matrix, Permutation
from . import _lib
from .sketch import (HADAMARD, build_composite, composite_sketch_right, members,
                     sketch_left_into, sketch_right_into, transform_kind_for_field)

logger = logging.getLogger(__name__)

MAX_RESAMPLES = 3        # randlu.py:46
STAGES = ("sketch1", "lu1", "sketch2", "pinv", "lu2")


@dataclass(frozen=True)
class RandLuParams:
    """randlu.py:49-95 (identical fields, defaults and invariants)."""

    r: int
    k1: int
    l1: int
    k2: int
    l2: int
    epsilon: float = 0.5
    delta: float = 0.1
    seed: int = 0
    field: str = REAL

    def __post_init__(self):
        if self.r < 1:
            raise ParameterError("target rank must be positive")
        if not self.r <= self.k1 <= self.k2:
            raise ParameterError(
                f"need r <= k1 <= k2, got r={self.r}, k1={self.k1}, k2={self.k2}")
        if not self.k1 < self.l1:
            raise ParameterError(f"need k1 < l1, got k1={self.k1}, l1={self.l1}")
        if not self.k2 < self.l2:
            raise ParameterError(f"need k2 < l2, got k2={self.k2}, l2={self.l2}")
        if not 0.0 < self.epsilon < 1.0:
            raise ParameterError("epsilon must lie in (0, 1)")
        if not 0.0 < self.delta < 1.0:
            raise ParameterError("delta must lie in (0, 1)")
        if self.field not in (REAL, COMPLEX):
            raise ParameterError(f"unknown field {self.field!r}")

    def check_against(self, m, n):
        if self.l1 > n:
            raise ParameterError(f"l1={self.l1} exceeds column count {n}")
        if self.l2 > m:
            raise ParameterError(f"l2={self.l2} exceeds row count {m}")
        if self.k2 > m:
            raise ParameterError(f"k2={self.k2} exceeds row count {m}")
        if self.k1 > m:
            raise ParameterError(f"k1={self.k1} exceeds row count {m}")


@dataclass
class RandLuResult:
    """randlu.py:98-114.  P, Q: host Permutations (device copies cached);
    L (m x k1), U (k1 x n): device Matrices.  ``elapsed`` in seconds."""

    P: Permutation
    Q: Permutation
    L: Matrix
    U: Matrix
    elapsed: dict = dc_field(default_factory=dict)
    attempt: int = 0
    extras: dict = dc_field(default_factory=dict)


def default_params(r, m, n, field=REAL, seed=0, mode="practical", epsilon=0.5,
                   delta=0.1) -> RandLuParams:
    """randlu.py:117-166 (practical and theoretical modes)."""
    if not 0.0 < epsilon < 1.0:
        raise ParameterError("epsilon must lie in (0, 1)")
    if not 0.0 < delta < 1.0:
        raise ParameterError("delta must lie in (0, 1)")
    if mode == "practical":
        if not 1 <= r <= min(m, n) / 2:
            raise ParameterError(f"need 1 <= r <= min(m,n)/2, got r={r} for {m} x {n}")
        k1 = min(n - 1, r + 8)
        k2 = min(m - 1, k1 + 8)
        l1 = min(n, 4 * k1)
        l2 = min(m, 4 * k2)
        if not r <= k1 < k2:
            raise ParameterError(
                f"degenerate size: clamped defaults collide (r={r}, k1={k1}, k2={k2} for {m} x {n})")
    elif mode == "theoretical":
        if not 1 <= r <= min(m, n):
            raise ParameterError(f"need 1 <= r <= min(m,n), got r={r}")
        re = r / epsilon
        k1 = max(r + 1, math.ceil(re * math.log(max(re, 2.0))))
        l1 = max(k1 + 1, math.ceil(r * r * math.log(max(re, 2.0)) ** 6 + re))
        l2 = math.ceil((r * r + r) / ((2 * epsilon - epsilon ** 2) ** 2 * delta))
        k2 = math.ceil(4.0 * (math.sqrt(r) + math.sqrt(8.0 * math.log(r * l2))) ** 2
                       * math.log(max(r, 2.0)))
        l1 = min(l1, n)
        l2 = min(l2, m)
        k1 = min(k1, l1 - 1, m)
        k2 = min(max(k2, k1), l2 - 1, m - 1)
        if not (r <= k1 <= k2 and k1 < l1 and k2 < l2):
            raise ParameterError(f"theoretical sizes do not fit a {m} x {n} matrix at r={r}")
    else:
        raise ParameterError(f"unknown mode {mode!r}")
    return RandLuParams(r=int(r), k1=int(k1), l1=int(l1), k2=int(k2), l2=int(l2),
                        epsilon=epsilon, delta=delta, seed=int(seed), field=field)


def params_from_north_star(m, n, k, l, width, seed=0) -> RandLuParams:
    """The (A, k, l, seed) form of BASELINE.json: r = k, k1 = l, l1 = width,
    k2 = min(m-1, k1+8), l2 = min(m, 4 k2) (the reference's practical rule,
    randlu.py:136-139) — SURVEY.md §0 finding 3."""
    k2 = min(m - 1, l + 8)
    return RandLuParams(r=k, k1=l, l1=width, k2=k2, l2=min(m, 4 * k2), seed=seed)


class _CompositeOps:
    """Structured sketch pair for one attempt (randlu.py:169-181)."""

    def __init__(self, params, m, n, seed1, seed2, device):
        kind = transform_kind_for_field(params.field)
        self.omega1 = build_composite(params.k1, params.l1, n, kind, seed1, device)
        self.omega2 = build_composite(params.k2, params.l2, m, kind, seed2, device)


def sparse_randomized_lu(a, params: RandLuParams, *, keep: bool = False) -> RandLuResult:
    """Randomized pivoted LU with structured projections (randlu.py:208-213).
    ``a``: Matrix, CUDA tensor (row-major fp32/fp64), numpy array or scipy
    sparse.  Deterministic: same inputs and params give bit-identical
    factors."""
    if not isinstance(a, Matrix):
        a = Matrix.from_device(a) if isinstance(a, torch.Tensor) and a.is_cuda else Matrix(a)
    return _pipeline(a, params, keep)


def gaussian_randomized_lu(a, params: RandLuParams, keep: bool = False) -> RandLuResult:
    """randlu.py:216-219: the same pipeline with dense Gaussian projections
    G1 (k1 x n) and G2 (k2 x m) applied by plain FP64 matrix products
    (randlu.py:184-205) — the paper's comparison baseline.  The draws are
    numpy's Philox(seed) standard normals (host, then uploaded: the ziggurat
    stream is kept bit-identical to the reference's); for dense A the three
    products run on the package's own FP64 tensor-core GEMM (srlu_dgemm, DMMA),
    for CSR A on cuSPARSE SpMM; the LUs, pseudo-inverse and rank test are the
    same kernels as the sparse path."""
    a = a if isinstance(a, Matrix) else Matrix(a)
    return _pipeline(a, params, keep, gaussian=True)


def _gaussian_host(k, n, seed):
    """randlu.py:197-205 (real field)."""
    g = np.random.Generator(np.random.Philox(seed))
    return g.standard_normal((k, n))


def _attempt_gaussian(a: Matrix, params: RandLuParams, attempt: int, keep: bool) -> RandLuResult:
    m, n = a.shape
    dev = a.device
    k1, k2 = params.k1, params.k2
    main = torch.cuda.current_stream(dev)
    ev = _stage_events(dev, len(STAGES) + 1)
    ev[0].record(main)
    g1 = torch.from_numpy(_gaussian_host(k1, n, params.seed + 2 * attempt)).to(dev)
    g2 = torch.from_numpy(_gaussian_host(k2, m, params.seed + 2 * attempt + 1)).to(dev)
    if a.is_sparse:
        indptr, indices, values = a.raw
        rows = torch.repeat_interleave(torch.arange(m, device=dev), indptr.diff())
        a_op = torch.sparse_coo_tensor(torch.stack([rows, indices.long()]), values.double(),
                                       (m, n), check_invariants=False).coalesce()
    else:
        a_op = a.raw.double() if a.raw.dtype != torch.float64 else a.raw
    if not bool(torch.isfinite(a_op.values() if a.is_sparse else a_op).all()):
        raise ValueError("matrix entries must be finite")
    if a.is_sparse:
        y = (a_op @ g1.t()).contiguous()                  # A . G1^T, m x k1 (SpMM)
    else:
        y = dgemm(a_op, g1.t().contiguous())
    ev[1].record(main)
    y_keep = y.clone() if keep else None
    perm, l1, _ = lu_row_pivot_dev(y)
    ev[2].record(main)
    red_lT = dgemm(l1.t().contiguous(), g2.t().contiguous())   # (G2 . L1)^T, k1 x k2
    g2p = torch.empty_like(g2)
    g2p[:, perm] = g2                                      # G2 . (P A) = G2p . A
    if a.is_sparse:
        red_aT = (a_op.t() @ g2p.t()).contiguous()        # (G2 P A)^T, n x k2 (SpMM)
    else:
        red_aT = dgemm(a_op.t().contiguous(), g2p.t().contiguous())
    ev[3].record(main)
    pinv_t, rank = pinv_dev(red_lT)
    core_t = dgemm(red_aT, pinv_t)
    ev[4].record(main)
    core_keep = core_t.clone() if keep else None
    q, lt, ut = lu_col_pivot_dev(core_t)
    l_final = dgemm(l1, lt, b_lower=True)
    ev[5].record(main)
    ev[5].synchronize()
    check_rank(rank.stats.cpu().numpy(), rank)
    elapsed = {name: ev[i].elapsed_time(ev[i + 1]) / 1e3 for i, name in enumerate(STAGES)}
    res = RandLuResult(P=Permutation(perm.cpu().numpy(), perm, validate=False),
                       Q=Permutation(q.cpu().numpy(), q, validate=False),
                       L=Matrix.from_device(l_final), U=_wrap(ut.t()), elapsed=elapsed,
                       attempt=attempt)
    if keep:
        res.extras = dict(Y=y_keep, L1=l1, red_l=red_lT.t(), red_a=red_aT.t(), pinv=pinv_t.t(),
                          core=core_keep.t(), Lt=lt, g1=g1, g2=g2)
    return res


def _pipeline(a: Matrix, params: RandLuParams, keep: bool, gaussian: bool = False) -> RandLuResult:
    m, n = a.shape
    params.check_against(m, n)
    if a.field != params.field:
        raise ParameterError(f"params.field={params.field} but matrix field is {a.field}")
    if params.field != REAL:
        raise NotImplementedError("complex128 field is out of scope of the B200 path")
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    last = None
    for attempt in range(1 + MAX_RESAMPLES):
        try:
            res = (_attempt_gaussian if gaussian else _attempt)(a, params, attempt, keep)
            t1 = torch.cuda.Event(enable_timing=True)
            t1.record()
            t1.synchronize()
            res.elapsed["total"] = t0.elapsed_time(t1) / 1e3
            return res
        except SingularMatrixError as err:
            last = err
            logger.warning("rank-deficient reduced system (attempt %d/%d, cond %.3e); "
                           "resampling sketches", attempt + 1, 1 + MAX_RESAMPLES, err.cond)
    raise DecompositionError(
        f"reduced system stayed rank deficient after {MAX_RESAMPLES} resamples "
        f"(last condition estimate {last.cond:.3e}); the sketch sizes "
        f"k2={params.k2}, l2={params.l2} are likely too small") from last


_SIDE_STREAMS = {}
_SMALL_A_BYTES = 256 << 20


_EVENTS = threading.local()


def _stage_events(dev, n):
    """Timing events of an attempt, created once per (thread, device) and
    re-recorded (their elapsed times are read before the attempt returns)."""
    key = torch.device(dev).index
    pool = getattr(_EVENTS, "pool", None)
    if pool is None:
        pool = _EVENTS.pool = {}
    evs = pool.get(key)
    if evs is None or len(evs) < n:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        pool[key] = evs
    return evs[:n]


def _side_stream(dev):
    key = torch.device(dev).index
    if key not in _SIDE_STREAMS:
        # high priority (testing knob SRLU_SIDE_PRIO=0 turns it off): the
        # side stream's small latency-bound kernels (Omega2 draws, QR/pinv,
        # rank test) take the next free SM slot ahead of the main stream's
        # queued CTAs instead of waiting for a whole streaming grid to drain
        prio = -1 if os.environ.get("SRLU_SIDE_PRIO", "1") != "0" else 0
        _SIDE_STREAMS[key] = torch.cuda.Stream(device=dev, priority=prio)
    return _SIDE_STREAMS[key]


def _pinned_copy(t: torch.Tensor) -> torch.Tensor:
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    return out


_NVTX = bool(os.environ.get("SRLU_NVTX"))


def _stage_mark(ev, i, stream):
    """Stage boundary i: the CUDA event behind ``elapsed`` and, with
    SRLU_NVTX=1, an NVTX range per stage (srlu.sketch1, srlu.lu1, ...) for
    timeline profilers."""
    ev[i].record(stream)
    if _NVTX:
        if i > 0:
            torch.cuda.nvtx.range_pop()
        if i < len(STAGES):
            torch.cuda.nvtx.range_push("srlu." + STAGES[i])


def _attempt(a: Matrix, params: RandLuParams, attempt: int, keep: bool) -> RandLuResult:
    """One pass of Algorithm 1 (randlu.py:246-276).  Two streams: the side
    stream draws Omega2 and builds its plan while K1/K2 run, and runs the
    small QR/pinv (K4) while K3 streams P·A on the main stream."""
    m, n = a.shape
    dev = a.device
    k1, k2 = params.k1, params.k2
    kind = transform_kind_for_field(params.field)
    main = torch.cuda.current_stream(dev)
    side = _side_stream(dev)
    ev = _stage_events(dev, len(STAGES) + 1)
    _stage_mark(ev, 0, main)

    y = torch.empty(m, k1, dtype=torch.float64, device=dev)
    if a.is_sparse:
        om1 = build_composite(k1, params.l1, n, kind, params.seed + 2 * attempt, dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        sketch_right_into(a, om1, y, flag)
    else:  # draws, plan, schedule and K1 in one C call
        flag = torch.empty(1, dtype=torch.int32, device=dev)
        om1 = composite_sketch_right(a, k1, params.l1, kind, params.seed + 2 * attempt, y, flag)
    _stage_mark(ev, 1, main)

    def omega2():
        # Omega2 (draws + plan + member table of L1) on the side stream,
        # independent of everything enqueued so far
        with torch.cuda.stream(side):
            om = build_composite(k2, params.l2, m, kind, params.seed + 2 * attempt + 1, dev)
            om.sem.plan()
            mem = members(om, None, 0, m, stream=side)
            e = torch.cuda.Event()
            e.record(side)
        return om, mem, e

    # A stream shorter than the host side of the Omega2 build (~0.15 ms):
    # enqueue K2 first so that it does not wait for that host work; longer
    # streams: Omega2 first, its device work overlapping K1
    small = not a.is_sparse and a.raw.numel() * a.raw.element_size() < _SMALL_A_BYTES
    if not small:
        om2, (mrow_l, msign_l, bptr2), ev_om2 = omega2()
    y_keep = y.clone() if keep else None
    perm, l1, _ = lu_row_pivot_dev(y)
    _stage_mark(ev, 2, main)
    if small:
        om2, (mrow_l, msign_l, bptr2), ev_om2 = omega2()

    # stage 2: Omega2 L1, then (K4 on the side stream) || Omega2 (P A)
    main.wait_event(ev_om2)
    for t in (om2.sem.row_of, om2.sem.sign, om2.fast.phase, om2.fast.sample_idx, mrow_l,
              msign_l, bptr2, *om2.sem.plan()):
        t.record_stream(main)
    red_lT = torch.empty(k1, k2, dtype=torch.float64, device=dev)
    sketch_left_into(Matrix.from_device(l1), om2, mrow_l, msign_l, bptr2, red_lT)
    ev_redl = torch.cuda.Event()
    ev_redl.record(main)
    side.wait_event(ev_redl)
    with torch.cuda.stream(side):
        # pinv first; the rank test follows on the side stream and overlaps
        # the core GEMM and K5 (only the final host decision needs it)
        pinv_t, rank, ev_pinv = pinv_dev(red_lT, stream=side, rank_event=True)
    pinv_t.record_stream(main)
    rank.record_stream(main)
    stats = rank.stats
    red_lT.record_stream(side)
    red_aT = torch.empty(n, k2, dtype=torch.float64, device=dev)
    if a.is_sparse:
        inv = torch.empty(m, dtype=torch.int32, device=dev)
        inv[perm] = torch.arange(m, dtype=torch.int32, device=dev)
        sketch_left_into(a, om2, None, None, None, red_aT, inv_perm=inv, flags=flag)
    else:
        mrow, msign, _ = members(om2, perm, 0, m)
        sketch_left_into(a, om2, mrow, msign, bptr2, red_aT)
    _stage_mark(ev, 3, main)

    main.wait_event(ev_pinv)
    core_t = dgemm(red_aT, pinv_t)      # (Omega2 P A)^T pinv^T = core^T, n x k1
    _stage_mark(ev, 4, main)
    core_keep = core_t.clone() if keep else None

    # one SM left to the side stream's rank test (a cooperative launch would
    # otherwise wait for it)
    q, lt, ut = lu_col_pivot_dev(core_t, reserve_sms=1)
    l_final = dgemm(l1, lt, b_lower=True)
    _stage_mark(ev, 5, main)

    # the one host sync of the attempt: rank test, non-finite flag, P, Q
    main.wait_stream(side)
    stats_h, flag_h, perm_h, q_h = (_pinned_copy(t) for t in (stats, flag, perm, q))
    ev[5].synchronize()
    torch.cuda.current_stream(dev).synchronize()
    fl = int(flag_h[0])
    if fl & 1:
        raise ValueError("matrix entries must be finite")
    if fl & 2:
        raise NotImplementedError("sketch_left_csr: a (column, bucket) group exceeds 8192 nonzeros")
    stats_host = check_rank(stats_h.numpy(), rank)
    elapsed = {name: ev[i].elapsed_time(ev[i + 1]) / 1e3 for i, name in enumerate(STAGES)}
    res = RandLuResult(P=Permutation(perm_h.numpy(), perm, validate=False),
                       Q=Permutation(q_h.numpy(), q, validate=False),
                       L=Matrix.from_device(l_final), U=_wrap(ut.t()), elapsed=elapsed,
                       attempt=attempt)
    if keep:
        res.extras = dict(Y=y_keep, L1=l1, red_l=red_lT.t(), red_a=red_aT.t(), pinv=pinv_t.t(),
                          stats=stats_host,
                          core=core_keep.t(), Lt=lt, omega1=om1, omega2=om2)
    return res


def _wrap(t: torch.Tensor) -> Matrix:
    """Wrap a (possibly column-major) device tensor as a Matrix without a copy."""
    mm = object.__new__(Matrix)
    mm._dense = t
    mm._indptr = mm._indices = mm._values = None
    mm.rows, mm.cols = int(t.shape[0]), int(t.shape[1])
    return mm


def approximation_error(a, res: RandLuResult) -> float:
    """||L U - P A Q||_F (randlu.py:279-302) on the device: K7
    (srlu_lu_error_dense / _csr), the L·(U Q^T) tiles on the FP64 tensor
    cores with P·A subtracted and squared in the epilogue; a fixed summation
    order (deterministic).  Evaluation only (never timed)."""
    if not isinstance(a, Matrix):
        a = Matrix.from_device(a) if isinstance(a, torch.Tensor) and a.is_cuda else Matrix(a)
    m, n = a.shape
    if res.L.rows != m or res.U.cols != n or res.L.cols != res.U.rows \
            or res.P.size != m or res.Q.size != n:
        raise ShapeError(f"factors {res.L.shape} x {res.U.shape} do not match target {a.shape}")
    lib = _lib.lib()
    dev = a.device
    k = res.L.cols
    perm = res.P.device_indices(dev)
    cols = res.Q.device_indices(dev)
    ld = res.L.to_dense().to(torch.float64)
    ld = ld if ld.stride(1) == 1 else ld.contiguous()
    ut = res.U.to_dense().to(torch.float64).t()        # n x k (U^T)
    ut = ut if ut.stride(1) == 1 else ut.contiguous()
    ws = _lib.workspace(lib.srlu_lu_error_workspace(m, n, k), dev)
    sq = torch.empty(1, dtype=torch.float64, device=dev)
    sh = _lib.stream_handle()
    if a.is_sparse:
        indptr, indices, vals = a.raw
        _lib.check(lib.srlu_lu_error_csr(_lib.ptr(ld), ld.stride(0), _lib.ptr(ut), ut.stride(0),
                                         _lib.ptr(perm), _lib.ptr(cols), _lib.ptr(indptr),
                                         _lib.ptr(indices), _lib.ptr(vals),
                                         _lib.dtype_code(vals.dtype), m, n, k, _lib.ptr(sq),
                                         _lib.ptr(ws), ws.numel(), sh), "lu_error")
    else:
        t = a.raw
        _lib.check(lib.srlu_lu_error_dense(_lib.ptr(ld), ld.stride(0), _lib.ptr(ut), ut.stride(0),
                                           _lib.ptr(perm), _lib.ptr(cols), _lib.ptr(t),
                                           _lib.dtype_code(t.dtype), m, n, t.stride(0), k,
                                           _lib.ptr(sq), _lib.ptr(ws), ws.numel(), sh),
                   "lu_error")
    return math.sqrt(float(sq.item()))
