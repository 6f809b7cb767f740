"""Row-sharded multi-GPU sparse randomized LU.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  A is
split into contiguous row shards; rank g owns rows [row0_g, row0_g+rows_g).
One attempt (reference randlu.py:246-276):

  stage 1  every rank: K0 draws (same seed -> same Omega1 everywhere) and
           K1 on its rows -> Y_g (rows_g x k1).  Rows of Y depend only on the
           same rows of A, so Y is bit-identical to the single-GPU Y.
  gather   Y_g -> rank 0 only (grouped point-to-point send/recv).
  lu1      rank 0: K2 -> P, L1; broadcast P (int64[m]).
  stage 2  every rank: Omega2 (same seed), member table restricted to its
           rows, K3 on its shard -> partial (Omega2 P A)^T_g (n x k2).
  pinv     rank 0 (while the ranks stream K3): Omega2 L1, K4 QR/pinv and the
           certified rank test; broadcast pinv^T (k2 x k1).
  core     every rank: core^T_g = partial_g . pinv^T (DMMA GEMM, 1/G of the
           core product each); NCCL reduce (SUM) of the n x k1 partials to
           rank 0 — pinv is linear, so sum(pinv . partial_g) = pinv . (Omega2
           P A); the cross-rank summation order differs from the sequential
           one (~1e-16 relative), so core is not bit-exact for world > 1.
  status   flags merged bit by bit (MAX over a 0/1 vector: bit 0 non-finite,
           bit 1 a CSR column beyond K3-CSR's limit) and the rank decision
           (factor.py:122-128, with the exact fallback) broadcast from rank 0:
           every rank raises or resamples in lockstep.
  tail     rank 0: K5 -> Q, L~, U; L = L1 L~ (the result lives on rank 0).

The per-rank compute is an injectable ``ops`` object: ``CudaOps`` (libsrlu
kernels, the product path) or, in tests, a numpy CPU stand-in
(tests/test_dist_gloo.py) — the sharding/collective logic is the same code.
"""

from __future__ import annotations

import json
import math
import os

import numpy as np
import torch
import torch.distributed as dist

from .errors import DecompositionError, SingularMatrixError
from .matrix import Matrix, Permutation
from .randlu import MAX_RESAMPLES, RandLuParams, RandLuResult, _wrap

FLAG_NONFINITE = 1
FLAG_LONG_COLUMN = 2


def shard_bounds(m: int, world: int, rank: int):
    """Contiguous, balanced row split: (row0, rows)."""
    base, rem = divmod(m, world)
    rows = base + (1 if rank < rem else 0)
    row0 = rank * base + min(rank, rem)
    return row0, rows


class CudaOps:
    """Per-rank compute with the libsrlu kernels (the product path)."""

    def __init__(self, device):
        self.device = torch.device(device)

    def sketch_right(self, a_local: Matrix, n, params, seed):
        from .sketch import build_composite, sketch_right_into
        om1 = build_composite(params.k1, params.l1, n, "hadamard", seed, self.device)
        y = torch.empty(a_local.rows, params.k1, dtype=torch.float64, device=self.device)
        flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        if a_local.rows > 0:
            sketch_right_into(a_local, om1, y, flag)
        return y, flag

    def lu_rows(self, y):
        from .factor import lu_row_pivot_dev
        perm, l1, _ = lu_row_pivot_dev(y)
        return perm, l1

    def omega2(self, m, params, seed):
        from .sketch import build_composite
        om2 = build_composite(params.k2, params.l2, m, "hadamard", seed, self.device)
        om2.sem.plan()
        return om2

    def sketch_left_partial(self, a_local: Matrix, row0, om2, perm, n, params, flag):
        from .sketch import members, sketch_left_into
        out = torch.zeros(n, params.k2, dtype=torch.float64, device=self.device)
        if a_local.rows == 0:
            return out
        if a_local.is_sparse:
            m = perm.numel()
            inv = torch.empty(m, dtype=torch.int32, device=self.device)
            inv[perm] = torch.arange(m, dtype=torch.int32, device=self.device)
            sketch_left_into(a_local, om2, None, None, None, out,
                             inv_perm=inv[row0:row0 + a_local.rows].contiguous(), flags=flag)
        else:
            mrow, msign, bptr = members(om2, perm, row0, a_local.rows)
            sketch_left_into(a_local, om2, mrow, msign, bptr, out)
        return out

    def pinv_async(self, l1, om2, params):
        """Omega2 L1 (K3 on L1), K4 QR/pinv + certified rank test (rank 0),
        on the side stream: they overlap this rank's K3 stream of P A."""
        from .factor import pinv_dev
        from .randlu import _side_stream
        from .sketch import members, sketch_left_into
        m, k1 = l1.shape
        main = torch.cuda.current_stream(self.device)
        side = _side_stream(self.device)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            mrow_l, msign_l, bptr2 = members(om2, None, 0, m)
            red_lT = torch.empty(k1, params.k2, dtype=torch.float64, device=self.device)
            sketch_left_into(Matrix.from_device(l1), om2, mrow_l, msign_l, bptr2, red_lT)
            pinv_t, rank_state = pinv_dev(red_lT)
        l1.record_stream(side)
        return pinv_t, rank_state, side

    def pinv_wait(self, handle):
        pinv_t, rank_state, side = handle
        main = torch.cuda.current_stream(self.device)
        main.wait_stream(side)
        pinv_t.record_stream(main)
        rank_state.record_stream(main)
        return pinv_t, rank_state

    def decide(self, rank_state):
        """factor.py:122-128 on rank 0: (singular, cond)."""
        from .factor import check_rank
        try:
            st = check_rank(rank_state.stats.cpu().numpy(), rank_state)
            return False, float(st[2])
        except SingularMatrixError as e:
            return True, float(e.cond)

    def gemm(self, a, b):
        from .factor import dgemm
        return dgemm(a, b)

    def tail(self, l1, core_t):
        from .factor import dgemm, lu_col_pivot_dev
        q, lt, ut = lu_col_pivot_dev(core_t)
        return q, dgemm(l1, lt, b_lower=True), ut


def _gather_rows_to_root(y_local, m, world, rank, group):
    """Y's row blocks -> rank 0 (grouped send/recv; rank 0 receives straight
    into its rows of Y).  Returns Y on rank 0, None elsewhere."""
    k = y_local.shape[1]
    if rank != 0:
        if y_local.shape[0]:
            dist.send(y_local.contiguous(), dst=0, group=group)
        return None
    y = torch.empty(m, k, dtype=y_local.dtype, device=y_local.device)
    _, rows0 = shard_bounds(m, world, 0)
    y[:rows0] = y_local
    ops = []
    for g in range(1, world):
        r0, rows = shard_bounds(m, world, g)
        if rows:
            ops.append(dist.P2POp(dist.irecv, y[r0:r0 + rows], g, group=group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return y


def _merge_flags(flag, dev, group):
    """Bit-wise OR across ranks (MAX per bit: a rank's non-finite bit is
    never masked by another rank's other bit)."""
    f = int(flag.item()) if isinstance(flag, torch.Tensor) else int(flag)
    bits = torch.tensor([1 if f & FLAG_NONFINITE else 0, 1 if f & FLAG_LONG_COLUMN else 0],
                        dtype=torch.int32, device=dev)
    dist.all_reduce(bits, op=dist.ReduceOp.MAX, group=group)
    return (FLAG_NONFINITE if int(bits[0]) else 0) | (FLAG_LONG_COLUMN if int(bits[1]) else 0)


DIST_STAGES = ("sketch1", "gather", "lu1", "sketch2", "core_reduce", "lu2")


def sparse_randomized_lu_dist(a_local: Matrix, m: int, params: RandLuParams, *, ops=None,
                              group=None, timings: dict | None = None) -> RandLuResult | None:
    """Row-sharded decomposition.  ``a_local``: this rank's contiguous row
    shard (rows shard_bounds(m, world, rank)) of the m x n matrix.  Returns
    the RandLuResult on rank 0 and None elsewhere; every rank raises the same
    error (non-finite input, unsupported CSR column, DecompositionError)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = a_local.cols
    row0, rows = shard_bounds(m, world, rank)
    if a_local.rows != rows:
        raise ValueError(f"rank {rank}: expected {rows} local rows, got {a_local.rows}")
    params.check_against(m, n)
    ops = ops if ops is not None else CudaOps(a_local.device)
    dev = ops.device
    k1, k2 = params.k1, params.k2
    last = None
    use_ev = timings is not None and dev.type == "cuda"
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(DIST_STAGES) + 1)] \
        if use_ev else None

    def mark(i):
        if evs is not None:
            evs[i].record()

    for attempt in range(1 + MAX_RESAMPLES):
        s1 = params.seed + 2 * attempt
        s2 = params.seed + 2 * attempt + 1
        mark(0)
        y_local, flag = ops.sketch_right(a_local, n, params, s1)
        mark(1)
        y = _gather_rows_to_root(y_local, m, world, rank, group)
        mark(2)
        om2 = ops.omega2(m, params, s2)
        rank_state = None
        if rank == 0:
            perm, l1 = ops.lu_rows(y)
            del y
        else:
            perm, l1 = torch.empty(m, dtype=torch.int64, device=dev), None
        dist.broadcast(perm, src=0, group=group)
        mark(3)
        if rank == 0:
            handle = ops.pinv_async(l1, om2, params)
        partial = ops.sketch_left_partial(a_local, row0, om2, perm, n, params, flag)
        mark(4)
        if rank == 0:
            pinv_t, rank_state = ops.pinv_wait(handle)
        else:
            pinv_t = torch.empty(k2, k1, dtype=torch.float64, device=dev)
        dist.broadcast(pinv_t, src=0, group=group)
        core_t = ops.gemm(partial, pinv_t)                 # n x k1 partial of core^T
        del partial
        dist.reduce(core_t, dst=0, op=dist.ReduceOp.SUM, group=group)
        mark(5)
        fl = _merge_flags(flag, dev, group)
        status = torch.zeros(2, dtype=torch.float64, device=dev)
        if rank == 0:
            singular, cond = ops.decide(rank_state)
            status[0] = 1.0 if singular else 0.0
            status[1] = cond
        dist.broadcast(status, src=0, group=group)
        if fl & FLAG_NONFINITE:
            raise ValueError("matrix entries must be finite")
        if fl & FLAG_LONG_COLUMN:
            raise NotImplementedError("sketch_left_csr: a column exceeds the supported length")
        if status[0].item():
            last = SingularMatrixError("rank-deficient reduced system", cond=float(status[1]))
            continue
        if rank != 0:
            return None
        q, l_final, ut = ops.tail(l1, core_t)
        if evs is not None:
            mark(6)
            evs[6].synchronize()
            timings.update({name: evs[i].elapsed_time(evs[i + 1]) for i, name in
                            enumerate(DIST_STAGES)})
        return RandLuResult(P=Permutation(perm.cpu().numpy(), perm, validate=False),
                            Q=Permutation(q.cpu().numpy(), q, validate=False),
                            L=Matrix.from_device(l_final),
                            U=_wrap(ut.t()), attempt=attempt)
    raise DecompositionError("reduced system stayed rank deficient after resampling") from last


# --------------------------------------------------------------------------
# bench.py --gpus N entry (one process per GPU under torchrun)


def bench_main(args, cfg, metric, workload, gen_config, time_region, flush_l2, ClockSampler,
               measured_peaks):
    """bench.py --gpus N: each rank generates only its row shard (the
    generators are seeded per 4096-row block, so the shards are the rows of
    the single-GPU matrix), then times K steps of sparse_randomized_lu_dist
    (barrier + synchronize around each, max over ranks)."""
    from . import _lib
    from .sketch import build_composite, sketch_right_into
    world = dist.get_world_size()
    rank = dist.get_rank()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    m, n = cfg["m"], cfg["n"]
    row0, rows = shard_bounds(m, world, rank)
    a, prm = gen_config(args.config, dev, row_range=(row0, row0 + rows))
    sparse = isinstance(a, tuple)
    if sparse:
        a_local = Matrix.from_csr(*a, shape=(rows, n))
    else:
        a_local = Matrix.from_device(a)
    local_bytes = sum(t.numel() * t.element_size() for t in a) if sparse else \
        a.numel() * a.element_size()
    tb = torch.tensor([float(local_bytes)], dtype=torch.float64, device=dev)
    dist.all_reduce(tb)
    nbytes = int(tb.item())
    params = RandLuParams(**prm)
    step = lambda: sparse_randomized_lu_dist(a_local, m, params)
    for _ in range(max(3, args.warmup)):
        step()
    _lib.LAUNCHES.reset()
    with ClockSampler(local) as clk:
        times = time_region(step, args.steps, barrier=dist.barrier)
    launches = _lib.LAUNCHES.total
    t = torch.tensor([float(np.mean(times))], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    timings = {}
    dist.barrier()
    sparse_randomized_lu_dist(a_local, m, params, timings=timings)

    # stage-1 stream (K1) of every rank's shard, timed alone, max over ranks
    om1 = build_composite(params.k1, params.l1, n, "hadamard", 0, dev)
    om1.sem.plan()
    y = torch.empty(rows, params.k1, dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    sketch_right_into(a_local, om1, y, flag)
    k1_ms = float(np.mean(time_region(lambda: sketch_right_into(a_local, om1, y, flag),
                                      args.steps, kernel=True)))
    tk = torch.tensor([k1_ms], device=dev)
    dist.all_reduce(tk, op=dist.ReduceOp.MAX)
    k1_ms = float(tk.item())
    k1_bytes = nbytes + m * params.k1 * 8

    # e2e: each rank's shard H2D from pinned host memory, the call, and the
    # D2H of P, Q, L, U on rank 0, inside the timed region
    host = tuple(x.cpu().pin_memory() for x in a) if sparse else a.cpu().pin_memory()
    d2h = {}

    def e2e_step():
        if sparse:
            dv = tuple(x.to(dev, non_blocking=True) for x in host)
            mat = Matrix.from_csr(*dv, shape=(rows, n))
        else:
            mat = Matrix.from_device(host.to(dev, non_blocking=True))
        r = sparse_randomized_lu_dist(mat, m, params)
        if r is not None:
            lh, uh = r.L.to_host(), r.U.to_host()
            d2h["bytes"] = lh.numel() * 8 + uh.numel() * 8 + (m + n) * 8

    e2e_step()
    e2e_times = time_region(e2e_step, min(args.steps, 5), barrier=dist.barrier)
    te = torch.tensor([float(np.mean(e2e_times))], device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    peak, peak_src = measured_peaks()
    if rank == 0:
        k1_gbs = k1_bytes / (k1_ms / 1e3) / 1e9
        line = {
            "metric": metric, "value": round(nbytes / (ms / 1e3) / 1e9, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded per 4096-row block, each rank generates its shard on "
                    "its device; BASELINE config shapes)",
            "config": {"workload": workload, "config_id": args.config, "m": m, "n": n,
                       "a_dtype": cfg["dtype"], "bytes_A": nbytes, "params": prm,
                       "parallelism": f"row-sharded x{world} (Y gathered to rank 0, P and "
                                      f"pinv broadcast, n x k1 core partials reduced)",
                       "l2": "flushed before every timed step"},
            "stages_ms": {k: round(v, 4) for k, v in timings.items()},
            "roofline": {"bound": "hbm", "kernel": "stage-1 sketch of every shard (K1), "
                                                   "max over ranks",
                         "achieved": round(k1_gbs, 1), "peak": peak * world, "unit": "GB/s",
                         "frac": round(k1_gbs / (peak * world), 4), "traffic": None,
                         "algorithmic_bytes": k1_bytes, "avg_launch_ms": round(k1_ms, 4),
                         "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs) x {world} GPUs"},
            "e2e": {"value": round(nbytes / (e2e_ms / 1e3) / 1e9, 3), "unit": "GB/s",
                    "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": d2h.get("bytes")},
            "cpu_baseline": None,
            "cpu_baseline_note": "reported by the N=1 run only (rank 0 at N=1)",
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
