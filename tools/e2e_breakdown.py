"""e2e step pieces (config 2): upload of A from pinned memory, the
decomposition, the result download — CUDA events on the current stream."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1601_04280_b200 as P
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
a, prm = bench.gen_config(c)
params = P.RandLuParams(**prm)
host_a = a.cpu().pin_memory()
for it in range(4):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    ev[0].record()
    dev = host_a.to("cuda", non_blocking=True)
    ev[1].record()
    mat = P.Matrix.from_device(dev)
    r = P.sparse_randomized_lu(mat, params)
    ev[2].record()
    lh = r.L.to_host(); uh = r.U.to_host()
    ev[3].record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    print(f"upload {ev[0].elapsed_time(ev[1]):.2f} ms  lu {ev[1].elapsed_time(ev[2]):.2f} ms  "
          f"download {ev[2].elapsed_time(ev[3]):.2f} ms  wall {wall:.2f} ms", flush=True)
