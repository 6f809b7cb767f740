"""Per-step wall times (CUDA events) of sparse_randomized_lu on a BASELINE
config, to find outlier steps: python tools/step_times.py CONFIG [STEPS]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1601_04280_b200 as P

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
a, prm = bench.gen_config(c)
A = bench.as_matrix(P, a, (bench.CONFIGS[c]["m"], bench.CONFIGS[c]["n"]))
params = P.RandLuParams(**prm)
for _ in range(3):
    P.sparse_randomized_lu(A, params)
torch.cuda.synchronize()
ts, hs, att = [], [], []
for _ in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    r = P.sparse_randomized_lu(A, params)
    e1.record()
    torch.cuda.synchronize()
    hs.append((time.perf_counter() - h0) * 1e3)
    ts.append(e0.elapsed_time(e1))
    att.append(r.attempt)
print("gpu ms", np.round(ts, 2).tolist())
print("host ms", np.round(hs, 2).tolist())
print("attempts", att)
print("allocator", torch.cuda.memory_stats().get("num_alloc_retries"), torch.cuda.memory_stats().get("num_device_alloc"))
