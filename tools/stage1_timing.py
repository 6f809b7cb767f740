"""GPU span of the Omega1 build (draws + plan) vs K1 inside sketch1 (config 2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1601_04280_b200 as P
from paper_1601_04280_b200.sketch import build_composite, sketch_right_into, transform_kind_for_field

a, prm = bench.gen_config(2)
A = P.Matrix.from_device(a)
params = P.RandLuParams(**prm)
kind = transform_kind_for_field(params.field)
res = []
for it in range(8):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record()
    om1 = build_composite(params.k1, params.l1, A.shape[1], kind, params.seed, A.device)
    e[1].record()
    e[2].record()
    y = torch.empty(A.shape[0], params.k1, dtype=torch.float64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    sketch_right_into(A, om1, y, flag)
    e[3].record()
    torch.cuda.synchronize()
    res.append([e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])])
r = np.median(np.array(res[2:]), axis=0) * 1e3
print("build_composite %.1f us  - %.1f  K1 (incl. y alloc) %.1f us" % tuple(r))

# host enqueue time of the one-call build
import time
hs = []
for it in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    om = build_composite(params.k1, params.l1, A.shape[1], kind, params.seed, A.device)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    hs.append([t1 - t0, t2 - t1])
h = np.median(np.array(hs[3:]), axis=0) * 1e6
print("host us: build_composite %.1f  then GPU drain %.1f" % tuple(h))
