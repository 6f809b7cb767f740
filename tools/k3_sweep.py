"""Time the stage-2 projection (K3) alone and its bucket-scatter part (K3a,
srlu_sem_scatter_dense) for a BASELINE config; the difference is K3b.
Settings as in k1_sweep.py (NAME=VAL,... or "-")."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1601_04280_b200 as P
from paper_1601_04280_b200 import _lib
from paper_1601_04280_b200.sketch import members, sketch_left_into

c = int(sys.argv[1])
a, prm = bench.gen_config(c)
cfg = bench.CONFIGS[c]
A = bench.as_matrix(P, a, (cfg["m"], cfg["n"]))
m, n = cfg["m"], cfg["n"]
nbytes = bench.a_bytes(a)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
om2 = P.build_composite(prm["k2"], prm["l2"], m, "hadamard", 1)
perm = torch.randperm(m, device="cuda")
mrow, msign, bptr = members(om2, perm, 0, m)
out = torch.empty(n, prm["k2"], dtype=torch.float64, device="cuda")
S = torch.empty(prm["l2"], n, dtype=torch.float64, device="cuda")
L = _lib.lib()
t = A.raw


def k3():
    sketch_left_into(A, om2, mrow, msign, bptr, out)


def k3a():
    _lib.check(L.srlu_sem_scatter_dense(_lib.ptr(t), _lib.dtype_code(t.dtype), m, n, t.stride(0),
                                        _lib.ptr(mrow), _lib.ptr(msign), _lib.ptr(bptr),
                                        prm["l2"], _lib.ptr(S), n, _lib.stream_handle()), "x")


def timeit(fn):
    fn()
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


ref = None
for setting in sys.argv[2:] or ["-"]:
    env = {}
    if setting != "-":
        for kv in setting.split(","):
            kk, v = kv.split("=")
            env[kk] = v
    for kk in [x for x in os.environ if x.startswith("SRLU_K3")]:
        del os.environ[kk]
    os.environ.update(env)
    t3 = timeit(k3)
    if ref is None:
        ref = out.clone()
    same = bool(torch.equal(out, ref))
    t3a = timeit(k3a)
    gbs = (nbytes + out.numel() * 8) / t3 / 1e6
    print(f"config {c} {setting:30s} K3 {t3:.4f} ms ({gbs:.0f} GB/s, frac {gbs / 6545:.3f})  "
          f"K3a {t3a:.4f} ms  K3b~{t3 - t3a:.4f} ms  same={same}", flush=True)
