"""The row-sharded path (dist.py) with the CUDA ops over NCCL at world size
1 on the single available B200: must reproduce the single-GPU factors
bit-for-bit (the reduce is the identity).  World sizes > 1 are covered by
tests/test_dist_gloo.py (host logic) — this box has one GPU."""

import os

import numpy as np
import pytest

from tests.conftest import cuda_ok

pytestmark = pytest.mark.gpu


def test_dist_world1_nccl_matches_single_gpu():
    if not cuda_ok():
        pytest.skip("needs a CUDA device")
    import torch
    import torch.distributed as dist
    import paper_1601_04280_b200 as P
    from paper_1601_04280_b200.dist import sparse_randomized_lu_dist
    from tests.golden.cases import gen_rank_noise
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        a = torch.tensor(gen_rank_noise(3000, 1500, 20, 1e-4, 3), device="cuda").float()
        prm = P.RandLuParams(r=20, k1=30, l1=120, k2=38, l2=152, seed=4)
        ref = P.sparse_randomized_lu(P.Matrix.from_device(a), prm)
        got = sparse_randomized_lu_dist(P.Matrix.from_device(a), a.shape[0], prm)
        np.testing.assert_array_equal(got.P.indices, ref.P.indices)
        np.testing.assert_array_equal(got.Q.indices, ref.Q.indices)
        np.testing.assert_array_equal(got.L.numpy(), ref.L.numpy())
        np.testing.assert_array_equal(got.U.numpy(), ref.U.numpy())
    finally:
        dist.destroy_process_group()
