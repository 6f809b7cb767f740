"""Time the stage-1 sketch kernel alone (CUDA events, L2 flushed) for a
BASELINE config under several SRLU_K1_* settings given as
NAME=VAL[,NAME=VAL] arguments ("-" = defaults).  Usage:
  python tools/k1_sweep.py 2 - SRLU_K1_RB=2 SRLU_K1_NOSCHED=1"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1601_04280_b200 as P
from paper_1601_04280_b200 import _lib
from paper_1601_04280_b200.sketch import sketch_right_into

c = int(sys.argv[1])
a, prm = bench.gen_config(c)
cfg = bench.CONFIGS[c]
A = bench.as_matrix(P, a, (cfg["m"], cfg["n"]))
nbytes = bench.a_bytes(a)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
y = torch.empty(cfg["m"], prm["k1"], dtype=torch.float64, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
ref = None
for setting in sys.argv[2:] or ["-"]:
    env = {}
    if setting != "-":
        for kv in setting.split(","):
            k, v = kv.split("=")
            env[k] = v
    for k in [k for k in os.environ if k.startswith("SRLU_K1_")]:
        del os.environ[k]
    os.environ.update(env)
    om = P.build_composite(prm["k1"], prm["l1"], cfg["n"], "hadamard", 0)
    sketch_right_into(A, om, y, flag)
    torch.cuda.synchronize()
    if ref is None:
        ref = y.clone()
    same = bool(torch.equal(y, ref))
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sketch_right_into(A, om, y, flag)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    info = (ctypes.c_int64 * 8)()
    L = _lib.lib()
    dcode = _lib.dtype_code(A.raw.dtype) if not A.is_sparse else 0
    L.srlu_k1_config(cfg["n"], prm["l1"], om.fast.pad, dcode, info)
    sched = [v for _, v in om.sem._sched if v is not None]
    words = int(sched[0][:4].view(torch.int32)[0].item()) if sched else 0
    geo = f"rb={info[0]} bpt={info[1]} c={info[2]} nch={info[3]} ns={info[4]} codes={words * 4 // 1024}KB/cap {info[5] // 1024}KB"
    gbs = (nbytes + y.numel() * 8) / ms / 1e6
    print(f"config {c} {setting:40s} {ms:8.4f} ms  {gbs:7.1f} GB/s  frac {gbs / 6545:.3f}  "
          f"same={same}  {geo}", flush=True)
