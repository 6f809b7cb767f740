"""Kernel timeline of one sparse_randomized_lu call (torch.profiler / CUPTI):
every kernel and memcpy with its start offset, duration and stream, plus the
GPU idle gaps (no kernel on any stream) longer than 2 us.  Usage:
  python tools/timeline.py CONFIG [OUT.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import bench
import paper_1601_04280_b200 as P

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
out = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/trace_c{c}.json"
a, prm = bench.gen_config(c)
cfg = bench.CONFIGS[c]
A = bench.as_matrix(P, a, (cfg["m"], cfg["n"]))
params = P.RandLuParams(**prm)
for _ in range(3):
    P.sparse_randomized_lu(A, params)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    res = P.sparse_randomized_lu(A, params)
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
ks = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
ks.sort(key=lambda e: e["ts"])
t0 = ks[0]["ts"]
print(f"config {c}: stages {dict((k, round(v * 1e3, 3)) for k, v in res.elapsed.items())}")
busy_end = t0
idle = 0.0
for e in ks:
    s, d = e["ts"], e["dur"]
    gap = s - busy_end
    if gap > 2:
        print(f"   -- idle {gap:8.1f} us")
        idle += gap
    name = e["name"].replace("void ", "")[:60]
    print(f"{s - t0:9.1f} {d:9.1f} us  s{e['args'].get('stream', '?'):<4} {name}")
    busy_end = max(busy_end, s + d)
print(f"span {busy_end - t0:.1f} us, idle (all streams) {idle:.1f} us, kernels {len(ks)}")
