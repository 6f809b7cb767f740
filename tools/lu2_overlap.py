"""Timing experiment: does the side-stream rank test delay the column LU?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import torch
from paper_1601_04280_b200 import _lib
from paper_1601_04280_b200 import RandLuParams
from paper_1601_04280_b200.randlu import sparse_randomized_lu

a, prm = bench.gen_config(2)
params = RandLuParams(**prm)
mode = sys.argv[1] if len(sys.argv) > 1 else "base"
if mode == "norank":
    import paper_1601_04280_b200.randlu as R
    L = _lib.lib()
    L.srlu_qr_rank = lambda *args: 0
    R.check_rank = lambda *args: None
for i in range(5):
    sparse_randomized_lu(a, params)
torch.cuda.synchronize()
import statistics
st = {}
for i in range(15):
    r = sparse_randomized_lu(a, params)
    for k, v in r.elapsed.items():
        st.setdefault(k, []).append(v)
print(mode, os.environ.get("SRLU_LU_MAX_GRID"), {k: round(statistics.median(v) * 1e3, 3) for k, v in st.items()})
