"""Host cost breakdown of build_composite on the GPU box."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1601_04280_b200 import _lib
from paper_1601_04280_b200.sketch import _STAGING
L = _lib.lib()
k, l, n = 110, 880, 16384
dev = torch.device("cuda")
def med(f, reps=200):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); ts.append(time.perf_counter() - t)
    return np.median(ts) * 1e6
ws_bytes = L.srlu_build_composite_workspace(n, l)
buf = torch.empty(1 << 22, dtype=torch.uint8, device=dev)
row_of = buf[0:n*4].view(torch.int32); sign = buf[1<<20:(1<<20)+n*8].view(torch.float64)
srt = buf[2<<20:(2<<20)+n*4].view(torch.int32); bptr = buf[3<<20:(3<<20)+(l+1)*4].view(torch.int32)
phase = buf[(3<<20)+8192:(3<<20)+8192+l*8].view(torch.float64); idx = buf[(3<<20)+32768:(3<<20)+32768+k*4].view(torch.int32)
wsb = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
st = torch.empty(L.srlu_build_composite_staging(k, l), dtype=torch.uint8, pin_memory=True)
padc = ctypes.c_int64(0)
sh = _lib.stream_handle()
def c_call():
    L.srlu_build_composite(0, k, l, n, _lib.ptr(row_of), _lib.ptr(sign), _lib.ptr(srt), _lib.ptr(bptr),
                           _lib.ptr(phase), _lib.ptr(idx), ctypes.addressof(padc), st.data_ptr(), st.numel(),
                           wsb.data_ptr(), ws_bytes, sh)
print("C build_composite call us %.1f" % med(c_call))
print("torch.empty device us %.1f" % med(lambda: torch.empty(300000, dtype=torch.uint8, device=dev)))
print("staging get+put us %.1f" % med(lambda: _STAGING.put(_STAGING.get(12000), torch.cuda.current_stream())))
print("6 views us %.1f" % med(lambda: [buf[i*1000:(i+1)*1000].view(torch.float64) for i in range(6)]))
print("stream_handle us %.1f" % med(lambda: _lib.stream_handle()))
def draws_only():
    ph = np.empty(l); i64 = np.empty(k, dtype=np.int64); p = np.zeros(1, dtype=np.int64)
    L.srlu_draw_fast_transform(2**32, k, l, ph.ctypes.data, i64.ctypes.data, p.ctypes.data)
print("host draws us %.1f" % med(draws_only))
