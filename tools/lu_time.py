"""Time lu_row_pivot_dev on random tall inputs (CUDA events, median of 5):
python tools/lu_time.py M K [M K ...]; SRLU_LU_* knobs apply."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1601_04280_b200.factor import lu_row_pivot_dev

args = [int(x) for x in sys.argv[1:]]
for m, k in zip(args[0::2], args[1::2]):
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    y = torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g)
    ts = []
    for _ in range(6):
        w = y.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = lu_row_pivot_dev(w)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    perm = out[0] if isinstance(out, (tuple, list)) else out
    h = int(torch.as_tensor(perm).double().cpu().numpy()[:64].dot(np.arange(64) + 1.0)) if torch.is_tensor(perm) else 0
    print(f"LU {m} x {k}: {np.median(ts[1:]):.3f} ms  (B2={os.environ.get('SRLU_LU_B2', 'default')}) perm-hash {h}")
