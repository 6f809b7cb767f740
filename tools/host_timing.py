"""Host wall time vs GPU span of sparse_randomized_lu (config 2)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_1601_04280_b200 as P
from bench import gen_config
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
a, prm = gen_config(c)
A = P.Matrix.from_device(a) if not isinstance(a, tuple) else P.Matrix.from_csr(*a, shape=(a[0].numel()-1, 65536))
params = P.RandLuParams(**prm)
for _ in range(3):
    P.sparse_randomized_lu(A, params)
torch.cuda.synchronize()
walls, gpus = [], []
for _ in range(10):
    t = time.perf_counter()
    r = P.sparse_randomized_lu(A, params)
    walls.append(time.perf_counter() - t)
    gpus.append(r.elapsed["total"])
print("wall ms", np.round(np.array(walls) * 1e3, 3))
print("gpu  ms", np.round(np.array(gpus) * 1e3, 3))
print("stages", {k: round(v * 1e3, 3) for k, v in r.elapsed.items()})
# host-only cost of the enqueue: time the launch phase without waiting (approx via profiler-free trick)
import cProfile, pstats, io
pr = cProfile.Profile(); pr.enable(); P.sparse_randomized_lu(A, params); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(15); print(s.getvalue()[:3000])
