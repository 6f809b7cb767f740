"""Time srlu_qr_pinv (QR + rank test + pinv) alone for the (k1, k2) of
configs 1, 2 and 4: the default (lookahead) QR against the shared-memory
dataflow one (SRLU_QR=smem) and the register-resident one (SRLU_QR=reg);
the pseudo-inverses must agree to round-off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1601_04280_b200.factor import pinv_dev


def timed(fn, n=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / n * 1e3


for k1, k2 in [(60, 68), (110, 118), (120, 128)]:
    g = torch.Generator(device="cuda").manual_seed(k1)
    mT = torch.randn(k1, k2, dtype=torch.float64, device="cuda", generator=g)
    res = {}
    for mode in ("la1", "la2", "la3", "la4", "smem"):
        os.environ["SRLU_QR"] = mode if mode == "smem" else "la"
        os.environ["SRLU_QR_DEPTH"] = mode[2:] if mode != "smem" else "2"
        us = timed(lambda: pinv_dev(mT))
        res[mode] = (us, pinv_dev(mT)[0].clone())
    os.environ.pop("SRLU_QR", None)
    ref = res["smem"][1]
    print(f"k1={k1} k2={k2}: " + ", ".join(
        f"{m} {us:7.1f} us (rel {float((p - ref).norm() / ref.norm()):.1e})" for m, (us, p) in res.items()))
