"""world_size-2 (gloo, CPU) test of the row-sharded orchestration in
paper_1601_04280_b200/dist.py: sharding, Y gather, P broadcast, partial
reduce, resample lockstep.  The per-rank compute is the CPU oracle (this is
the host logic test; the CUDA ops are covered by the gpu tests)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import draws, randlu as O


class OracleOps:
    device = torch.device("cpu")

    def sketch_right(self, a_local, n, params, seed):
        om1 = draws.build_composite(params.k1, params.l1, n, seed)
        y = O.apply_sketch_right(a_local.raw.numpy(), om1)
        return torch.from_numpy(np.ascontiguousarray(y)), torch.zeros(1, dtype=torch.int32)

    def lu_rows(self, y):
        perm, l1, _ = O.lu_row_pivot(y.numpy())
        return torch.from_numpy(perm.astype(np.int64)), torch.from_numpy(np.ascontiguousarray(l1))

    def omega2(self, m, params, seed):
        return draws.build_composite(params.k2, params.l2, m, seed)

    def sketch_left_partial(self, a_local, row0, om2, perm, n, params, flag):
        m = perm.numel()
        p = perm.numpy()
        loc = (p >= row0) & (p < row0 + a_local.rows)
        pa = np.zeros((m, n))
        pa[loc] = a_local.raw.numpy()[p[loc] - row0]
        red = O.apply_sketch_left(om2, pa)          # k2 x n
        return torch.from_numpy(np.ascontiguousarray(red.T))

    def pinv_async(self, l1, om2, params):
        red_l = O.apply_sketch_left(om2, l1.numpy())
        try:
            return torch.from_numpy(np.ascontiguousarray(O.left_pseudo_inverse(red_l).T)), None
        except O.SingularMatrixError as e:
            return torch.zeros(params.k2, params.k1, dtype=torch.float64), e

    def pinv_wait(self, handle):
        return handle

    def decide(self, state):
        return (True, state.cond) if state is not None else (False, 1.0)

    def gemm(self, a, b):
        return torch.from_numpy(np.ascontiguousarray(a.numpy() @ b.numpy()))

    def tail(self, l1, core_t):
        q, lt, u = O.lu_col_pivot(core_t.numpy().T)
        return (torch.from_numpy(q.astype(np.int64)), torch.from_numpy(O.matmul(l1.numpy(), lt)),
                torch.from_numpy(np.ascontiguousarray(u.T)))


class FlagOps(OracleOps):
    """Injects K1/K3 status bits on chosen ranks (non-finite entry in one
    shard, an over-long CSR column in another)."""

    def __init__(self, rank, nonfinite_rank=None, longcol_rank=None):
        self.rank, self.nf, self.lc = rank, nonfinite_rank, longcol_rank

    def sketch_right(self, a_local, n, params, seed):
        y, flag = super().sketch_right(a_local, n, params, seed)
        if self.rank == self.nf:
            flag[0] |= 1
        return y, flag

    def sketch_left_partial(self, a_local, row0, om2, perm, n, params, flag):
        if self.rank == self.lc:
            flag[0] |= 2
        return super().sketch_left_partial(a_local, row0, om2, perm, n, params, flag)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, a, prm, out, flags=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1601_04280_b200 import Matrix, RandLuParams
        from paper_1601_04280_b200.dist import shard_bounds, sparse_randomized_lu_dist
        m = a.shape[0]
        row0, rows = shard_bounds(m, world, rank)
        a_local = Matrix(np.ascontiguousarray(a[row0:row0 + rows]), device="cpu",
                         check_finite=False)
        ops = OracleOps() if flags is None else FlagOps(rank, **flags)
        try:
            res = sparse_randomized_lu_dist(a_local, m, RandLuParams(**prm), ops=ops)
        except (ValueError, NotImplementedError) as e:
            out.put((rank, type(e).__name__))
            return
        if rank == 0:
            out.put(dict(P=res.P.indices.copy(), Q=res.Q.indices.copy(),
                         L=res.L.raw.numpy().copy(), U=res.U.raw.numpy().copy(),
                         attempt=res.attempt))
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


def _run(world, a, prm, flags=None, nres=1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, a, prm, q, flags))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(nres)]
    res = res[0] if nres == 1 else res
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return res


def test_shard_bounds_cover_rows():
    from paper_1601_04280_b200.dist import shard_bounds
    for m in (1, 7, 100, 16384, 1048577):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(m, w, r) for r in range(w)]
            assert spans[0][0] == 0
            assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert spans[-1][0] + spans[-1][1] == m
            assert max(s[1] for s in spans) - min(s[1] for s in spans) <= 1


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_matches_single_process(world):
    from tests.golden.cases import gen_rank_noise
    a = gen_rank_noise(301, 170, 8, 1e-3, 4)
    prm = dict(r=8, k1=16, l1=64, k2=24, l2=96, seed=9)
    got = _run(world, a, prm)
    ref = O.sparse_randomized_lu(a, prm)
    np.testing.assert_array_equal(got["P"], ref["P"])       # Y rows are shard-local: exact
    np.testing.assert_array_equal(got["Q"], ref["Q"])
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
    assert rel(got["L"], ref["L"]) <= 1e-10
    assert rel(got["U"], ref["U"]) <= 1e-10


def test_row_sharded_resample_lockstep():
    from tests.golden import cases
    a, prm = cases.pipeline_cases()["lowrank_resample"]
    got = _run(2, a, prm)
    assert got["attempt"] == 2


@pytest.mark.parametrize("flags,expect", [
    (dict(nonfinite_rank=1, longcol_rank=0), "ValueError"),      # bit 0 not masked by bit 1
    (dict(nonfinite_rank=None, longcol_rank=1), "NotImplementedError"),
    (dict(nonfinite_rank=2, longcol_rank=None), "ValueError"),
])
def test_status_bits_merged_bitwise_all_ranks_raise(flags, expect):
    """dist.py merges the K1/K3 status bits per bit (MAX of 0/1 vectors):
    a non-finite entry in one shard and an over-long CSR column in another
    both reach every rank, and every rank raises the same error."""
    from tests.golden.cases import gen_rank_noise
    a = gen_rank_noise(240, 150, 6, 1e-3, 2)
    prm = dict(r=6, k1=12, l1=48, k2=20, l2=80, seed=1)
    got = _run(3, a, prm, flags=flags, nres=3)
    assert sorted(r for r, _ in got) == [0, 1, 2]
    assert all(name == expect for _, name in got), got
