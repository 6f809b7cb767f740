"""Per-step phase timing of the LU kernel (CTA 0 clock64 trace)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1601_04280_b200 as P
from paper_1601_04280_b200 import _lib
from paper_1601_04280_b200.factor import lu_row_pivot_dev, lu_col_pivot_dev
L = _lib.lib()
HAS_DBG = hasattr(L, "srlu_lu_debug_trace")
if HAS_DBG: L.srlu_lu_debug_trace.argtypes = [ctypes.c_void_p]
for name, (M, k), fn in [("row 16384x110", (16384, 110), lu_row_pivot_dev), ("col 16384x110", (16384, 110), lu_col_pivot_dev),
                         ("row 262144x220", (262144, 220), lu_row_pivot_dev)]:
    dbg = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
    y = torch.randn(M, k, dtype=torch.float64, device="cuda")
    fn(y.clone()); torch.cuda.synchronize()
    if HAS_DBG: L.srlu_lu_debug_trace(ctypes.c_void_p(dbg.data_ptr()))
    yc = y.clone()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); fn(yc); e.record(); e.synchronize()
    if not HAS_DBG:
        print(f"{name}: {s.elapsed_time(e)*1e3/k:.2f} us/step total")
        continue
    L.srlu_lu_debug_trace(ctypes.c_void_p(0))
    t = dbg.view(4096, 8)[:k, :5].cpu().numpy().astype(np.float64)
    d = np.diff(t, axis=1)
    nxt = t[1:, 0] - t[:-1, 4]
    print(f"{name}: {s.elapsed_time(e)*1e3/k:.2f} us/step total; cycles/step: A->pub {d[:,0].mean():.0f}  pub->barrier {d[:,1].mean():.0f}  barrier->winner {d[:,2].mean():.0f}  winner->end {d[:,3].mean():.0f}  end->nextA {nxt.mean():.0f}  (step span {np.diff(t[:,0]).mean():.0f})")
