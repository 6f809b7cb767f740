"""The paper's comparison on one B200: sparse (CountSketch + SRHT) vs dense
Gaussian sketches in the same pipeline, wall time per decomposition (CUDA
events, L2 flushed, mean of 10 after 3 warm-ups) and ||LU - PAQ||_F.
python tools/gauss_vs_sparse.py CONFIG"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import numpy as np
import torch
import bench
import paper_1601_04280_b200 as P

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
a, prm = bench.gen_config(c)
cfg = bench.CONFIGS[c]
A = bench.as_matrix(P, a, (cfg["m"], cfg["n"]))
params = P.RandLuParams(**prm)
out = {"config": c}
for name, fn in (("sparse", P.sparse_randomized_lu), ("gaussian", P.gaussian_randomized_lu)):
    for _ in range(3):
        r = fn(A, params)
    ts = bench.time_region(lambda: fn(A, params), 10)
    r = fn(A, params)
    out[name] = {"ms": round(float(np.mean(ts)), 3),
                 "stages_ms": {k: round(v * 1e3, 3) for k, v in r.elapsed.items()},
                 "err": P.approximation_error(A, r)}
print(json.dumps(out))
