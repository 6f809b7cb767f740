"""cProfile of the host side of stage 1 (composite_sketch_right) at a config."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1601_04280_b200 as P
from paper_1601_04280_b200.sketch import composite_sketch_right

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
a, prm = bench.gen_config(c)
cfg = bench.CONFIGS[c]
A = bench.as_matrix(P, a, (cfg["m"], cfg["n"]))
y = torch.empty(cfg["m"], prm["k1"], dtype=torch.float64, device="cuda")
flag = torch.empty(1, dtype=torch.int32, device="cuda")
def one(seed):
    return composite_sketch_right(A, prm["k1"], prm["l1"], "hadamard", seed, y, flag)
for i in range(5):
    one(i); torch.cuda.synchronize()
ts = []
for i in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); one(i % 3); ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
ts.sort()
print(f"host time of composite_sketch_right: median {ts[len(ts)//2]*1e6:.1f} us, min {ts[0]*1e6:.1f} us")
pr = cProfile.Profile()
for i in range(200):
    torch.cuda.synchronize()
    pr.enable(); one(i % 3); pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(18)
