"""One config-N decomposition inside cudaProfilerStart/Stop (for
`ncu --profile-from-start off`): warm up, then profile exactly one call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1601_04280_b200 as P

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
a, prm = bench.gen_config(c)
A = bench.as_matrix(P, a, (bench.CONFIGS[c]["m"], bench.CONFIGS[c]["n"]))
params = P.RandLuParams(**prm)
for _ in range(3):
    P.sparse_randomized_lu(A, params)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
r = P.sparse_randomized_lu(A, params)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print({k: round(v * 1e3, 3) for k, v in r.elapsed.items()})
