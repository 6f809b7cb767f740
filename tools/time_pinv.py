import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1601_04280_b200 import _lib
from paper_1601_04280_b200.factor import pinv_dev, dgemm
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize(); return s.elapsed_time(e) / n
for k1, k2, n in [(110, 118, 16384), (220, 228, 8192), (550, 558, 65536)]:
    mT = torch.randn(k1, k2, dtype=torch.float64, device="cuda")
    M = mT.t().contiguous()
    ra = torch.randn(n, k2, dtype=torch.float64, device="cuda")
    print(k1, k2, "pinv_dev %.3f ms" % t(lambda: pinv_dev(mT)),
          "torch.qr %.3f ms" % t(lambda: torch.linalg.qr(M)),
          "dgemm core %.3f ms" % t(lambda: dgemm(ra, torch.randn(k2, k1, dtype=torch.float64, device='cuda'))),
          "torch mm %.3f ms" % t(lambda: ra @ torch.randn(k2, k1, dtype=torch.float64, device='cuda')))
    qf, rf = torch.linalg.qr(M); rf = rf.contiguous(); rft = rf.t().contiguous()
    stats = torch.empty(4, dtype=torch.float64, device="cuda")
    L = _lib.lib()
    print("   rank_estimate %.3f ms" % t(lambda: L.srlu_rank_estimate(_lib.ptr(rf), k1, rf.stride(0), _lib.ptr(rft), rft.stride(0), _lib.ptr(stats), _lib.stream_handle())),
          "solve_tri %.3f ms" % t(lambda: torch.linalg.solve_triangular(rf, qf.t().contiguous(), upper=True)))
