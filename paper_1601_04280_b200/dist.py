"""Row-sharded multi-GPU sparse randomized LU.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  A is
split into contiguous row shards; rank g owns rows [row0_g, row0_g+rows_g).

  stage 1  every rank: K0 draws (same seed -> same Omega1 everywhere) and
           K1 on its rows -> Y_g (rows_g x k1).  Rows of Y depend only on the
           same rows of A, so Y is bit-identical to the single-GPU Y.
  gather   Y_g -> rank 0 (all_gather of row-padded blocks).
  lu1      rank 0: K2 -> P, L1.  broadcast P (int64[m]).
  stage 2  every rank: Omega2 (same seed), member table restricted to its
           rows, K3 on its shard -> partial (Omega2 P A)^T (n x k2).  The
           FWHT and subsample are linear, so partials are reduced after them.
  reduce   partials -> rank 0 (NCCL reduce, SUM).  The cross-rank summation
           order differs from the sequential one, so Omega2·P·A (hence core)
           is no longer bit-exact for world > 1 (~1e-16 relative).
  tail     rank 0: Omega2 L1, pinv, core, K5, L = L1 L~.  The resample
           decision is broadcast so all ranks retry in lockstep.

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

    def tail(self, l1, om2, red_aT, params):
        from .factor import dgemm, lu_col_pivot_dev, pinv_dev
        from .sketch import members, sketch_left_into
        m, k1 = l1.shape
        mrow_l, msign_l, bptr2 = members(om2, None, 0, m)
        red_lT = torch.empty(k1, params.k2, dtype=torch.float64, device=self.device)
        sketch_left_into(Matrix.from_device(l1), om2, mrow_l, msign_l, bptr2, red_lT)
        pinv_t, stats = pinv_dev(red_lT)
        core_t = dgemm(red_aT, pinv_t)
        q, lt, ut = lu_col_pivot_dev(core_t)
        l_final = dgemm(l1, lt, b_lower=True)
        return q, l_final, ut, stats


def _gather_rows(y_local, m, world, rank, group):
    """Gather the row blocks of Y onto every rank (row-padded all_gather);
    only rank 0 uses the result."""
    rows_max = math.ceil(m / world)
    k = y_local.shape[1]
    buf = torch.zeros(rows_max, k, dtype=y_local.dtype, device=y_local.device)
    buf[:y_local.shape[0]] = y_local
    out = torch.empty(world * rows_max, k, dtype=y_local.dtype, device=y_local.device)
    try:
        dist.all_gather_into_tensor(out, buf, group=group)
    except (RuntimeError, NotImplementedError):  # backends without the fused form (gloo)
        dist.all_gather(list(out.chunk(world)), buf, group=group)
    if rank != 0:
        return None
    parts = []
    for g in range(world):
        _, rows = shard_bounds(m, world, g)
        parts.append(out[g * rows_max:g * rows_max + rows])
    return torch.cat(parts, 0).contiguous()


def sparse_randomized_lu_dist(a_local: Matrix, m: int, params: RandLuParams, *, ops=None,
                              group=None) -> RandLuResult | None:
    """Row-sharded decomposition.  ``a_local``: this rank's contiguous row
    shard (rows shard_bounds(m, world, rank)) of the m x n matrix.  Returns
    the RandLuResult on rank 0 and None elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = a_local.cols
    row0, rows = shard_bounds(m, world, rank)
    if a_local.rows != rows:
        raise ValueError(f"rank {rank}: expected {rows} local rows, got {a_local.rows}")
    params.check_against(m, n)
    ops = ops if ops is not None else CudaOps(a_local.device)
    dev = ops.device
    last = None
    for attempt in range(1 + MAX_RESAMPLES):
        s1 = params.seed + 2 * attempt
        s2 = params.seed + 2 * attempt + 1
        y_local, flag = ops.sketch_right(a_local, n, params, s1)
        y = _gather_rows(y_local, m, world, rank, group)
        if rank == 0:
            perm, l1 = ops.lu_rows(y)
        else:
            perm, l1 = torch.empty(m, dtype=torch.int64, device=dev), None
        dist.broadcast(perm, src=0, group=group)
        om2 = ops.omega2(m, params, s2)
        partial = ops.sketch_left_partial(a_local, row0, om2, perm, n, params, flag)
        dist.reduce(partial, dst=0, op=dist.ReduceOp.SUM, group=group)
        # status: [nonfinite flag (any rank), singular flag, cond]
        fl = flag.to(torch.float64)
        dist.all_reduce(fl, op=dist.ReduceOp.MAX, group=group)
        status = torch.zeros(3, dtype=torch.float64, device=dev)
        result = None
        if rank == 0:
            q, l_final, ut, stats = ops.tail(l1, om2, partial, params)
            st = stats.cpu().numpy() if isinstance(stats, torch.Tensor) else np.asarray(stats)
            status[1] = float(st[3])
            status[2] = float(st[2]) if st[1] > 0 else float("inf")
            result = (perm, q, l_final, ut)
        status[0] = fl[0]
        dist.broadcast(status, src=0, group=group)
        if int(status[0].item()) & 1:
            raise ValueError("matrix entries must be finite")
        if status[1].item():
            last = SingularMatrixError("rank-deficient reduced system", cond=float(status[2]))
            continue
        if rank != 0:
            return None
        perm, q, l_final, ut = result
        return RandLuResult(P=Permutation(perm.cpu().numpy(), perm, validate=False),
                            Q=Permutation(q.cpu().numpy(), q, validate=False),
                            L=Matrix.from_device(l_final),
                            U=_wrap(ut.t()), attempt=attempt)
    raise DecompositionError("reduced system stayed rank deficient after resampling") from last


# --------------------------------------------------------------------------
# bench.py --gpus N entry (one process per GPU under torchrun)


def bench_main(args, cfg, metric, workload, gen_config, time_region, flush_l2, ClockSampler,
               measured_peaks):
    world = dist.get_world_size()
    rank = dist.get_rank()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    m, n = cfg["m"], cfg["n"]
    a, prm = gen_config(args.config, dev)
    row0, rows = shard_bounds(m, world, rank)
    if isinstance(a, tuple):
        indptr, indices, vals = a
        p0, p1 = int(indptr[row0]), int(indptr[row0 + rows])
        a_local = Matrix.from_csr(indptr[row0:row0 + rows + 1] - p0, indices[p0:p1],
                                  vals[p0:p1], (rows, n))
        nbytes = sum(t.numel() * t.element_size() for t in a)
    else:
        a_local = Matrix.from_device(a[row0:row0 + rows].contiguous())
        nbytes = a.numel() * a.element_size()
        del a
    params = RandLuParams(**prm)
    step = lambda: sparse_randomized_lu_dist(a_local, m, params)
    for _ in range(max(3, args.warmup)):
        step()
    with ClockSampler(local) as clk:
        times = time_region(step, args.steps, barrier=dist.barrier)
    t = torch.tensor([float(np.mean(times))], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0:
        line = {
            "metric": metric, "value": round(nbytes / (ms / 1e3) / 1e9, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, generated on device; BASELINE config shapes)",
            "config": {"workload": workload, "config_id": args.config, "m": m, "n": n,
                       "bytes_A": nbytes, "params": prm,
                       "parallelism": f"row-sharded x{world} (NCCL gather Y, reduce partials)",
                       "l2": "flushed before every timed step"},
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
