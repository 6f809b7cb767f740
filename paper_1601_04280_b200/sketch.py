"""Random projection operators on the device (the reference's sketch.py).

Draws (K0) are bit-exact with the reference's numpy ``Generator(Philox)``
streams (sketch.py:42-43, :103-114, :214-235, :269-278): the sparse
embedding's n bucket/sign draws are generated on the GPU, the transform
stage's l phases + Fisher-Yates permutation of ``pad`` items on the host
(C, inside libsrlu).  Application runs the fused CUDA kernels K1 (right
sketch, stage 1) and K3 (left sketch, stage 2).  Only the real64 /
Walsh-Hadamard field is on the B200 path (every BASELINE config is real).
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _lib
from .errors import ParameterError, ShapeError
from .matrix import COMPLEX, REAL, Matrix, _default_device

STAGE_SEED_OFFSET = 1 << 32      # sketch.py:36
FOURIER = "fourier"
HADAMARD = "hadamard"


def _next_pow2(n):
    return 1 << (int(n) - 1).bit_length()


def transform_kind_for_field(field):
    """sketch.py:50-57"""
    if field == REAL:
        return HADAMARD
    if field == COMPLEX:
        return FOURIER
    raise ParameterError(f"unknown field {field!r}")


def _check_seed(seed):
    seed = int(seed)
    if seed < 0 or seed >= 1 << 64:
        raise ParameterError(f"seed must lie in [0, 2**64), got {seed}")
    return seed


@dataclass(frozen=True, eq=False)
class SparseEmbedding:
    """k x n sparse sign embedding (sketch.py:60-100): column j has the
    single entry sign[j] in row row_of[j].  Device arrays; the bucket-sorted
    plan (sorted sources, bucket pointers) is built once, lazily."""

    out_dim: int
    in_dim: int
    row_of: torch.Tensor   # int32 [in_dim]
    sign: torch.Tensor     # float64 [in_dim], +-1
    seed: int = 0
    _plan: list = dc_field(default_factory=list, repr=False)
    _sched: list = dc_field(default_factory=list, repr=False)

    @property
    def shape(self):
        return (self.out_dim, self.in_dim)

    def plan(self, stream=None):
        """(sorted int32[n] with sign in bit 31, bucket_ptr int32[l+1])."""
        if not self._plan:
            L = _lib.lib()
            dev = self.row_of.device
            srt = torch.empty(self.in_dim, dtype=torch.int32, device=dev)
            bptr = torch.empty(self.out_dim + 1, dtype=torch.int32, device=dev)
            ws = _lib.workspace(L.srlu_sem_plan_workspace(self.in_dim, self.out_dim), dev)
            _lib.check(L.srlu_sem_plan(_lib.ptr(self.row_of), _lib.ptr(self.sign), self.in_dim,
                                       self.out_dim, _lib.ptr(srt), _lib.ptr(bptr),
                                       _lib.ptr(ws), ws.numel(), _lib.stream_handle(stream)),
                       "sem_plan")
            self._plan.extend([srt, bptr])
        return self._plan[0], self._plan[1]

    def k1_schedule(self, dtype_code, pad, stream=None):
        """Gather schedule of the scheduled K1 kernel (srlu_k1_schedule) for
        an A of this element type, built once per (dtype, pad) on `stream`;
        None when the shape is outside that kernel's range."""
        key = ("k1s", dtype_code, pad)
        for k_, v in self._sched:
            if k_ == key:
                return v
        L = _lib.lib()
        nbytes = L.srlu_k1_schedule_bytes(self.in_dim, self.out_dim, pad, dtype_code)
        buf = None
        if nbytes:
            srt, bptr = self.plan(stream)
            buf = torch.empty(nbytes, dtype=torch.uint8, device=srt.device)
            _lib.check(L.srlu_k1_schedule(_lib.ptr(srt), _lib.ptr(bptr), self.in_dim, self.out_dim,
                                          pad, dtype_code, _lib.ptr(buf), nbytes,
                                          _lib.stream_handle(stream)),
                       "k1_schedule" if _k1_grouped(L, self.in_dim, self.out_dim, pad, dtype_code)
                       else "k1_schedule_1")
        self._sched.append((key, buf))
        return buf

    def row_counts(self):
        return torch.bincount(self.row_of.long(), minlength=self.out_dim)


def _k1_grouped(L, n, l, pad, dtype_code) -> bool:
    """Whether the K1 schedule for this shape runs the group-sort kernel
    (several bucket slots per lane)."""
    info = (ctypes.c_int64 * 8)()
    L.srlu_k1_config(n, l, pad, dtype_code, info)
    return info[1] >= 2


def build_sem(k, n, seed, device=None) -> SparseEmbedding:
    """Draw a k x n sparse sign embedding on the device (sketch.py:103-114)."""
    if not 1 <= k <= n:
        raise ParameterError(f"need 1 <= k <= n, got k={k}, n={n}")
    seed = _check_seed(seed)
    L = _lib.lib()
    dev = torch.device(device) if device is not None else _default_device()
    row_of = torch.empty(n, dtype=torch.int32, device=dev)
    sign = torch.empty(n, dtype=torch.float64, device=dev)
    ws = _lib.workspace(L.srlu_draw_sem_workspace(n, k), dev)
    _lib.check(L.srlu_draw_sem(seed, k, n, _lib.ptr(row_of), _lib.ptr(sign), _lib.ptr(ws),
                               ws.numel(), _lib.stream_handle()), "build_sem")
    return SparseEmbedding(int(k), int(n), row_of, sign, seed=seed)


@dataclass(frozen=True, eq=False)
class FastTransformSketch:
    """k x l subsampled Walsh-Hadamard transform (sketch.py:143-201):
    scale * Sample(H_pad/sqrt(pad) · diag(phase) x)."""

    out_dim: int
    in_dim: int
    phase: torch.Tensor        # float64 [in_dim], +-1 (device)
    sample_idx: torch.Tensor   # int32 [out_dim] (device)
    pad: int
    scale: float
    kind: str = HADAMARD
    seed: int = 0
    phase_host: np.ndarray = None
    sample_idx_host: np.ndarray = None

    @property
    def shape(self):
        return (self.out_dim, self.in_dim)

    @property
    def field(self):
        return REAL

    @property
    def mult(self):
        # sketch.py:330 / :345: scale / sqrt(pad), one fp64 multiply per output
        return self.scale / math.sqrt(self.pad)


def build_fast_transform(k, l, kind, seed, device=None) -> FastTransformSketch:
    """Draw a k x l subsampled fast transform (sketch.py:214-235)."""
    if kind not in (FOURIER, HADAMARD):
        raise ParameterError(f"unknown transform kind {kind!r}")
    if kind == FOURIER:
        raise NotImplementedError("the complex128 / FFT lane is out of scope of the B200 path")
    if l < 1:
        raise ParameterError(f"need l >= 1, got {l}")
    pad = _next_pow2(l)
    if not 1 <= k <= pad:
        raise ParameterError(f"need 1 <= k <= {pad}, got k={k}")
    seed = _check_seed(seed)
    L = _lib.load()
    pin = torch.cuda.is_available()
    phase_t = torch.empty(l, dtype=torch.float64, pin_memory=pin)
    idx_t = torch.empty(k, dtype=torch.int64, pin_memory=pin)
    padc = np.zeros(1, dtype=np.int64)
    _lib.check(L.srlu_draw_fast_transform(seed, k, l, phase_t.data_ptr(), idx_t.data_ptr(),
                                          padc.ctypes.data), "build_fast_transform")
    assert int(padc[0]) == pad
    phase, idx = phase_t.numpy(), idx_t.numpy()
    dev = torch.device(device) if device is not None else _default_device()
    phase_d = phase_t.to(dev, non_blocking=True)
    idx_d = idx_t.to(dev, non_blocking=True).to(torch.int32)
    return FastTransformSketch(int(k), int(l), phase_d, idx_d, pad, math.sqrt(pad / k), kind,
                               seed=seed, phase_host=phase, sample_idx_host=idx)


@dataclass(frozen=True, eq=False)
class CompositeSketch:
    """sketch.py:238-266: sparse stage followed by the transform stage."""

    sem: SparseEmbedding
    fast: FastTransformSketch

    def __post_init__(self):
        if self.fast.in_dim != self.sem.out_dim:
            raise ShapeError("stage mismatch between embedding and transform")

    @property
    def out_dim(self):
        return self.fast.out_dim

    @property
    def in_dim(self):
        return self.sem.in_dim

    @property
    def shape(self):
        return (self.out_dim, self.in_dim)


class _StagingPool:
    """Pinned host staging buffers for the transform-stage draws, reused
    once the upload that last read them has completed (event-guarded)."""

    def __init__(self):
        self._free = []  # (nbytes, pinned uint8 tensor, event)

    def get(self, nbytes):
        for i, (nb, buf, ev) in enumerate(self._free):
            if nb >= nbytes and ev.query():
                del self._free[i]
                return buf
        return torch.empty(max(nbytes, 4096), dtype=torch.uint8, pin_memory=True)

    def put(self, buf, stream):
        ev = torch.cuda.Event()
        ev.record(stream)
        self._free.append((buf.numel(), buf, ev))
        if len(self._free) > 8:
            self._free.pop(0)


_STAGING = _StagingPool()


_LAYOUTS = {}


def _composite_layout(L, k, l, n, k1_dtype):
    """Byte layout of one composite sketch (+ optional K1 schedule) in a
    single device buffer; cached per shape."""
    # the kernel-selection knobs change the schedule's size: part of the key
    env = os.environ
    key = (k, l, n, k1_dtype, env.get("SRLU_K1_TMEM"), env.get("SRLU_K1_NOSCHED"),
           env.get("SRLU_K1_STAGE"), env.get("SRLU_K1_RB"))
    lay = _LAYOUTS.get(key)
    if lay is None:
        i4 = lambda c: ((c * 4 + 7) // 8) * 8
        # phase and idx adjacent: the C side uploads both in one copy
        off = {"sign": 0, "phase": n * 8}
        off["idx"] = off["phase"] + l * 8
        off["row"] = off["idx"] + i4(k)
        off["sorted"] = off["row"] + i4(n)
        off["bptr"] = off["sorted"] + i4(n)
        off["ws"] = ((off["bptr"] + i4(l + 1)) + 255) // 256 * 256
        ws_bytes = L.srlu_build_composite_workspace(n, l)
        sched_bytes = 0
        if k1_dtype is not None:
            sched_bytes = L.srlu_k1_schedule_bytes(n, l, _next_pow2(l), k1_dtype)
        off["sched"] = (off["ws"] + ws_bytes + 255) // 256 * 256
        total = off["sched"] + max(sched_bytes, 0)
        # the schedule builder's extra group-sort kernel runs only for
        # multi-slot lanes (srlu_k1_config info[1] = buckets per lane >= 2)
        off["grouped"] = bool(sched_bytes) and _k1_grouped(L, n, l, _next_pow2(l), k1_dtype)
        lay = (off, ws_bytes, sched_bytes, total, L.srlu_build_composite_staging(k, l))
        _LAYOUTS[key] = lay
    return lay


def build_composite(k, l, n, kind, seed, device=None, stream=None, k1_dtype=None) -> CompositeSketch:
    """sketch.py:269-278 (transform stage seeded seed + 2**32), in one C-ABI
    call: device sparse draws and the accumulation plan, then host transform
    draws -> pinned staging -> upload, all enqueued on `stream`; with
    ``k1_dtype`` (an A element-type code) also the scheduled K1's gather
    schedule.  The device work is enqueued before the Python bookkeeping."""
    return _composite(k, l, n, kind, seed, device, stream, k1_dtype, None)


def composite_sketch_right(a: Matrix, k, l, kind, seed, y: torch.Tensor, nonfinite: torch.Tensor,
                           stream=None) -> CompositeSketch:
    """Stage 1 of an attempt for a dense A (randlu.py:252-253): build_composite
    (k x n, `seed`) and y = A · omega^* with nonfinite reset to 0 first, in ONE
    C call (srlu_composite_sketch_right_dense) so that K1 is enqueued right
    behind the draws and its schedule; the Python bookkeeping of the sketch
    object runs while K1 streams A."""
    t = a.raw
    n = a.cols
    es = t.element_size()
    aligned = t.data_ptr() % 16 == 0 and (t.stride(0) * es) % 16 == 0 and (n * es) % 16 == 0
    k1_dtype = _lib.dtype_code(t.dtype)
    return _composite(k, l, n, kind, seed, t.device, stream, k1_dtype if aligned else None,
                      (t, k1_dtype, y, nonfinite))


# Sketch cache.  A composite sketch depends only on
# (k, l, n, kind, seed) — not on A — so repeated decompositions with the same
# parameters can reuse the draws, the bucket plan and the K1 schedule.  OFF by
# default: the reference redraws on every call (randlu.py:250-251) and
# bench.py times that work; enable with set_sketch_cache(True) or
# SRLU_SKETCH_CACHE=1.  Entries hold device buffers (LRU, 8 by default).
_CACHE = {"on": bool(os.environ.get("SRLU_SKETCH_CACHE")), "max": 8, "lock": threading.Lock(),
          "map": {}, "hits": 0, "misses": 0}


def set_sketch_cache(enabled: bool, max_entries: int = 8) -> None:
    """Turn the composite-sketch cache on or off (off drops the entries)."""
    with _CACHE["lock"]:
        _CACHE["on"] = bool(enabled)
        _CACHE["max"] = max(1, int(max_entries))
        if not enabled:
            _CACHE["map"].clear()


def sketch_cache_stats() -> dict:
    with _CACHE["lock"]:
        return {"enabled": _CACHE["on"], "entries": len(_CACHE["map"]), "hits": _CACHE["hits"],
                "misses": _CACHE["misses"]}


def _composite(k, l, n, kind, seed, device, stream, k1_dtype, right):
    if not _CACHE["on"]:
        return _composite_build(k, l, n, kind, seed, device, stream, k1_dtype, right)
    dev = torch.device(device) if device is not None else _default_device()
    key = (int(k), int(l), int(n), kind, int(seed), dev.index if dev.index is not None else
           torch.cuda.current_device(), k1_dtype)
    with _CACHE["lock"]:
        hit = _CACHE["map"].pop(key, None)
        if hit is not None:
            _CACHE["map"][key] = hit          # most recently used last
            _CACHE["hits"] += 1
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    if hit is not None:
        om, ev = hit
        s.wait_event(ev)                      # the draws were enqueued on another stream
        if right is not None:                 # the fused call's K1, on the cached sketch
            t, _, y, nonfinite = right
            with torch.cuda.stream(s):
                nonfinite.zero_()
            sketch_right_into(Matrix.from_device(t), om, y, nonfinite, stream=stream)
        return om
    om = _composite_build(k, l, n, kind, seed, device, stream, k1_dtype, right)
    ev = torch.cuda.Event()
    ev.record(s)
    with _CACHE["lock"]:
        _CACHE["misses"] += 1
        _CACHE["map"][key] = (om, ev)
        while len(_CACHE["map"]) > _CACHE["max"]:
            _CACHE["map"].pop(next(iter(_CACHE["map"])))
    return om


def _composite_build(k, l, n, kind, seed, device, stream, k1_dtype, right):
    if kind not in (FOURIER, HADAMARD):
        raise ParameterError(f"unknown transform kind {kind!r}")
    if kind == FOURIER:
        raise NotImplementedError("the complex128 / FFT lane is out of scope of the B200 path")
    if not 1 <= l <= n:
        raise ParameterError(f"need 1 <= k <= n, got k={l}, n={n}")
    pad = _next_pow2(l)
    if not 1 <= k <= pad:
        raise ParameterError(f"need 1 <= k <= {pad}, got k={k}")
    seed = _check_seed(seed)
    L = _lib.lib()
    dev = torch.device(device) if device is not None else _default_device()
    off, ws_bytes, sched_bytes, total, st_bytes = _composite_layout(L, k, l, n, k1_dtype)
    buf = torch.empty(total, dtype=torch.uint8, device=dev)
    base = buf.data_ptr()
    staging = _STAGING.get(st_bytes)
    padc = ctypes.c_int64(0)
    cur = stream if stream is not None else torch.cuda.current_stream(dev)   # looked up once
    sh = ctypes.c_void_p(cur.cuda_stream)
    P_ = ctypes.c_void_p
    if right is None:
        _lib.check(L.srlu_build_composite_k1(
            seed, k, l, n, P_(base + off["row"]), P_(base + off["sign"]), P_(base + off["sorted"]),
            P_(base + off["bptr"]), P_(base + off["phase"]), P_(base + off["idx"]),
            ctypes.addressof(padc), staging.data_ptr(), staging.numel(), P_(base + off["ws"]),
            ws_bytes, -1 if k1_dtype is None else k1_dtype,
            P_(base + off["sched"]) if sched_bytes else None, sched_bytes, sh),
            ("build_composite_k1_g" if off["grouped"] else "build_composite_k1") if sched_bytes
            else "build_composite")
    else:
        t, dcode, y, nonfinite = right
        m = t.shape[0]
        _lib.check(L.srlu_composite_sketch_right_dense(
            seed, k, l, n, P_(base + off["row"]), P_(base + off["sign"]), P_(base + off["sorted"]),
            P_(base + off["bptr"]), P_(base + off["phase"]), P_(base + off["idx"]),
            ctypes.addressof(padc), staging.data_ptr(), staging.numel(), P_(base + off["ws"]),
            ws_bytes, P_(base + off["sched"]) if sched_bytes else None, sched_bytes,
            P_(t.data_ptr()), dcode, m, t.stride(0), math.sqrt(pad / k) / math.sqrt(pad),
            P_(y.data_ptr()),
            y.stride(0), P_(nonfinite.data_ptr()), sh),
            ("composite_sketch_right_dense_g" if off["grouped"] else "composite_sketch_right_dense")
            if sched_bytes else "composite_sketch_right_dense_nosched")
    _STAGING.put(staging, cur)
    assert padc.value == pad
    isz = {torch.float64: 8, torch.int32: 4}
    view = lambda o, cnt, dt: buf[off[o]:off[o] + cnt * isz[dt]].view(dt)
    sem = SparseEmbedding(int(l), int(n), view("row", n, torch.int32),
                          view("sign", n, torch.float64), seed=seed)
    sem._plan.extend([view("sorted", n, torch.int32), view("bptr", l + 1, torch.int32)])
    if k1_dtype is not None:
        sem._sched.append((("k1s", k1_dtype, pad),
                           buf[off["sched"]:off["sched"] + sched_bytes] if sched_bytes else None))
    fast = FastTransformSketch(int(k), int(l), view("phase", l, torch.float64),
                               view("idx", k, torch.int32), pad, math.sqrt(pad / k), kind,
                               seed=seed + STAGE_SEED_OFFSET)
    return CompositeSketch(sem, fast)


# ---------------------------------------------------------------------------
# application


def _as_matrix(a):
    return a if isinstance(a, Matrix) else Matrix(a)


def sketch_right_into(a: Matrix, omega: CompositeSketch, y: torch.Tensor, nonfinite: torch.Tensor,
                      stream=None):
    """K1: y (m x k, fp64, row-major) = A · omega^*; nonfinite |= flag."""
    L = _lib.lib()
    sem, fast = omega.sem, omega.fast
    m, n = a.shape
    sh = _lib.stream_handle(stream)
    if a.is_sparse:
        indptr, indices, vals = a.raw
        _lib.check(L.srlu_sketch_right_csr(
            _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(vals), _lib.dtype_code(vals.dtype),
            m, n, _lib.ptr(sem.row_of), _lib.ptr(sem.sign), sem.out_dim, _lib.ptr(fast.phase),
            _lib.ptr(fast.sample_idx), fast.out_dim, fast.pad, fast.mult, _lib.ptr(y),
            y.stride(0), _lib.ptr(nonfinite), sh), "sketch_right_csr")
    else:
        t = a.raw
        dcode = _lib.dtype_code(t.dtype)
        es = t.element_size()
        aligned = t.data_ptr() % 16 == 0 and (t.stride(0) * es) % 16 == 0 and (n * es) % 16 == 0
        sched = sem.k1_schedule(dcode, fast.pad, stream) if aligned else None
        if sched is not None:
            _lib.check(L.srlu_sketch_right_dense_sched(
                _lib.ptr(t), dcode, m, n, t.stride(0), _lib.ptr(sched), sched.numel(),
                sem.out_dim, _lib.ptr(fast.phase), _lib.ptr(fast.sample_idx), fast.out_dim,
                fast.pad, fast.mult, _lib.ptr(y), y.stride(0), _lib.ptr(nonfinite), sh),
                "sketch_right_dense_sched")
            return
        srt, bptr = sem.plan()
        _lib.check(L.srlu_sketch_right_dense(
            _lib.ptr(t), _lib.dtype_code(t.dtype), m, n, t.stride(0), _lib.ptr(srt),
            _lib.ptr(bptr), sem.out_dim, _lib.ptr(fast.phase), _lib.ptr(fast.sample_idx),
            fast.out_dim, fast.pad, fast.mult, _lib.ptr(y), y.stride(0), _lib.ptr(nonfinite),
            sh), "sketch_right_dense")


def apply_sketch_right(a, omega: CompositeSketch) -> Matrix:
    """``a @ omega^*`` (sketch.py:362-368), one fused kernel."""
    a = _as_matrix(a)
    if omega.in_dim != a.cols:
        raise ShapeError(f"sketch expects {omega.in_dim} columns, got {a.cols}")
    y = torch.empty(a.rows, omega.out_dim, dtype=torch.float64, device=a.device)
    flag = torch.zeros(1, dtype=torch.int32, device=a.device)
    sketch_right_into(a, omega, y, flag)
    if int(flag.item()):
        raise ValueError("matrix entries must be finite")
    return Matrix.from_device(y)


def members(omega2: CompositeSketch, perm: torch.Tensor | None, row0: int, rows: int,
            stream=None):
    """Member table of the left sketch restricted to local rows [row0, row0+rows)."""
    L = _lib.lib()
    sem = omega2.sem
    srt, bptr = sem.plan(stream)
    m = sem.in_dim
    mrow = torch.empty(m, dtype=torch.int32, device=srt.device)
    msign = torch.empty(m, dtype=torch.float64, device=srt.device)
    _lib.check(L.srlu_sem_members(_lib.ptr(srt), m, _lib.ptr(perm), row0, rows, _lib.ptr(mrow),
                                  _lib.ptr(msign), _lib.stream_handle(stream)), "sem_members")
    return mrow, msign, bptr


def sketch_left_into(a: Matrix, omega2: CompositeSketch, mrow, msign, bptr, outT: torch.Tensor,
                     inv_perm=None, flags=None, stream=None):
    """K3: outT (cols x k2) = (omega2 · P a)^T over a's (local) rows.
    CSR: ``flags`` (int32 device scalar) gets bit 2 if a column is too long."""
    L = _lib.lib()
    fast = omega2.fast
    sh = _lib.stream_handle(stream)
    if a.is_sparse:
        indptr, indices, vals = a.raw
        nnz = vals.numel()
        ws = _lib.workspace(L.srlu_sketch_left_csr_workspace(a.rows, a.cols, nnz,
                                                             omega2.sem.out_dim, fast.pad),
                            a.device)
        _lib.check(L.srlu_sketch_left_csr(
            _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(vals), _lib.dtype_code(vals.dtype),
            a.rows, a.cols, nnz, _lib.ptr(inv_perm), _lib.ptr(omega2.sem.row_of),
            _lib.ptr(omega2.sem.sign), omega2.sem.out_dim, _lib.ptr(fast.phase),
            _lib.ptr(fast.sample_idx), fast.out_dim, fast.pad, fast.mult, _lib.ptr(outT),
            outT.stride(0), _lib.ptr(ws), ws.numel(), _lib.ptr(flags), sh),
            # launch accounting: banded count + scan and the tiled column scan
            # (n >= 8192, counters in shared memory) add three kernels
            "sketch_left_csr_big" if 8192 <= a.cols <= 102400 else "sketch_left_csr")
        return
    t = a.raw
    ws = _lib.workspace(L.srlu_sketch_left_workspace(a.cols, omega2.sem.out_dim, fast.pad),
                        a.device)
    _lib.check(L.srlu_sketch_left_dense(
        _lib.ptr(t), _lib.dtype_code(t.dtype), a.rows, a.cols, t.stride(0), _lib.ptr(mrow),
        _lib.ptr(msign), _lib.ptr(bptr), omega2.sem.out_dim, _lib.ptr(fast.phase),
        _lib.ptr(fast.sample_idx), fast.out_dim, fast.pad, fast.mult, _lib.ptr(outT),
        outT.stride(0), _lib.ptr(ws), ws.numel(), sh), "sketch_left_dense")


def apply_sketch_left(omega: CompositeSketch, a, perm=None) -> Matrix:
    """``omega @ (P a)`` (sketch.py:371-378; P = identity when perm is None).
    Returns the k x cols product (a transposed view of the kernel's
    cols x k output)."""
    a = _as_matrix(a)
    if omega.in_dim != a.rows:
        raise ShapeError(f"sketch expects {omega.in_dim} rows, got {a.rows}")
    pd = None
    if perm is not None:
        pd = perm.device_indices(a.device) if hasattr(perm, "device_indices") else perm
    outT = torch.empty(a.cols, omega.out_dim, dtype=torch.float64, device=a.device)
    if a.is_sparse:
        inv = None
        if pd is not None:
            inv = torch.empty(a.rows, dtype=torch.int32, device=a.device)
            inv[pd] = torch.arange(a.rows, dtype=torch.int32, device=a.device)
        else:
            inv = torch.arange(a.rows, dtype=torch.int32, device=a.device)
        flags = torch.zeros(1, dtype=torch.int32, device=a.device)
        sketch_left_into(a, omega, None, None, None, outT, inv_perm=inv, flags=flags)
        if int(flags.item()) & 2:
            raise NotImplementedError("sketch_left_csr: a (column, bucket) group exceeds 8192 nonzeros")
    else:
        mrow, msign, bptr = members(omega, pd, 0, a.rows)
        sketch_left_into(a, omega, mrow, msign, bptr, outT)
    return Matrix.from_device(outT.t())
