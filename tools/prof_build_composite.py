import sys, time, cProfile, pstats, io
sys.path.insert(0, '/root/repo')
import torch
import paper_1601_04280_b200 as P
from paper_1601_04280_b200.sketch import build_composite
for _ in range(5): build_composite(110, 880, 16384, "hadamard", 0, "cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for i in range(200): om = build_composite(110, 880, 16384, "hadamard", i, "cuda")
torch.cuda.synchronize()
print("per call ms", (time.perf_counter() - t) / 200 * 1e3)
pr = cProfile.Profile(); pr.enable()
for i in range(200): om = build_composite(110, 880, 16384, "hadamard", i, "cuda")
pr.disable(); torch.cuda.synchronize()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(20); print(s.getvalue()[:4000])
