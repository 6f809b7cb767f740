"""Run sparse_randomized_lu on a BASELINE config a few times (for ncu launch
lists: the last call's launches are one decomposition).  Usage:
  python tools/one_decomp.py CONFIG [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1601_04280_b200 as P

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
a, prm = bench.gen_config(c)
cfg = bench.CONFIGS[c]
A = bench.as_matrix(P, a, (cfg["m"], cfg["n"]))
torch.cuda.synchronize()
for _ in range(reps):
    P.sparse_randomized_lu(A, P.RandLuParams(**prm))
torch.cuda.synchronize()
print("ok")
