"""Stage-1 breakdown (config N): host enqueue time and GPU span of the
composite draws+plan, the K1 gather schedule and K1 itself, as in _attempt."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1601_04280_b200 as P
from paper_1601_04280_b200.sketch import build_composite, sketch_right_into

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
a, prm = bench.gen_config(c)
cfg = bench.CONFIGS[c]
A = bench.as_matrix(P, a, (cfg["m"], cfg["n"]))
y = torch.empty(cfg["m"], prm["k1"], dtype=torch.float64, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
rows = []
for it in range(8):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    h0 = time.perf_counter()
    ev[0].record()
    om = build_composite(prm["k1"], prm["l1"], cfg["n"], "hadamard", it, "cuda",
                         k1_dtype=None if A.is_sparse else P._lib.dtype_code(A.raw.dtype))
    h1 = time.perf_counter()
    ev[1].record()
    h2 = time.perf_counter()
    ev[2].record()
    sketch_right_into(A, om, y, flag)
    h3 = time.perf_counter()
    ev[3].record()
    torch.cuda.synchronize()
    rows.append([(h1 - h0) * 1e3, (h2 - h1) * 1e3, (h3 - h2) * 1e3,
                 ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])])
r = np.median(np.array(rows[2:]), axis=0)
print(f"config {c}: host ms composite+sched {r[0]:.3f} - {r[1]:.3f} k1-call {r[2]:.3f} | "
      f"gpu ms composite {r[3]:.3f} sched {r[4]:.3f} k1 {r[5]:.3f}")
