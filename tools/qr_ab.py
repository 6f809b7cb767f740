"""pinv_dev timing per QR variant (SRLU_QR = smem | reg | cluster) at the configs' (k1, k2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1601_04280_b200.factor import pinv_dev

def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize(); return s.elapsed_time(e) / n

for k1, k2 in [(60, 68), (110, 118), (120, 128), (220, 228), (550, 558)]:
    g = torch.Generator(device="cuda"); g.manual_seed(k1)
    mT = torch.randn(k1, k2, dtype=torch.float64, device="cuda", generator=g)
    try:
        print(os.environ.get("SRLU_QR", "default"), k1, k2, "pinv_dev %.3f ms" % t(lambda: pinv_dev(mT)))
    except Exception as ex:
        print(os.environ.get("SRLU_QR", "default"), k1, k2, "ERR", str(ex)[:80])
