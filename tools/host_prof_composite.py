import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import bench
import paper_1601_04280_b200 as P
from paper_1601_04280_b200 import _lib, sketch as S
c = 2
a, prm = bench.gen_config(c)
cfg = bench.CONFIGS[c]
A = bench.as_matrix(P, a, (cfg["m"], cfg["n"]))
L = _lib.lib()
orig = L.srlu_build_composite_k1
tc = []
def wrapped(*args):
    t = time.perf_counter(); r = orig(*args); tc.append(time.perf_counter() - t); return r
class LW:
    def __getattr__(self, k): return wrapped if k == "srlu_build_composite_k1" else getattr(L, k)
S._lib.lib = lambda: LW()
dc = _lib.dtype_code(A.raw.dtype)
tb, ty, tk = [], [], []
for it in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    om = S.build_composite(prm["k1"], prm["l1"], cfg["n"], "hadamard", it % 3, "cuda", k1_dtype=dc)
    t1 = time.perf_counter()
    y = torch.empty(cfg["m"], prm["k1"], dtype=torch.float64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    t2 = time.perf_counter()
    S.sketch_right_into(A, om, y, flag)
    t3 = time.perf_counter()
    tb.append(t1 - t0); ty.append(t2 - t1); tk.append(t3 - t2)
    torch.cuda.synchronize()
md = lambda v: f"{np.median(v[5:]) * 1e6:.1f} us"
print("build_composite", md(tb), "of which C call", md(tc), "| empty+zeros", md(ty), "| sketch_right_into", md(tk))
# C-level pieces
import ctypes
