"""Diagnostic: where does the GPU tail (pinv, core, L~, U) sit relative to
the reference and to the extended-precision answer?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from threadpoolctl import threadpool_limits
from oracle import randlu as O
import paper_1601_04280_b200 as P
from tests.golden.cases import gen_rank_noise, pipeline_cases


def rel(x, y):
    return float(np.linalg.norm(np.asarray(x) - np.asarray(y)) / np.linalg.norm(y))


def run(name, a, prm):
    with threadpool_limits(1):
        ref = O.sparse_randomized_lu(a, prm, keep=True)
    qx, Lx, Ux = O.forward_error_band(ref["red_l"], ref["red_a"], ref["L1"])
    res = P.sparse_randomized_lu(a, P.RandLuParams(**prm), keep=True)
    ex = res.extras
    core_g = ex["core"].cpu().numpy()
    pinv_g = ex["pinv"].cpu().numpy()
    # variants on the GPU from the (bit-exact) red_l, red_a
    M = torch.tensor(ref["red_l"], device="cuda")
    RA = torch.tensor(ref["red_a"], device="cuda")
    q_, r_ = torch.linalg.qr(M)
    core_solve = torch.linalg.solve_triangular(r_, q_.t() @ RA, upper=True).cpu().numpy()
    pinv_cpu_core_gpu = (torch.tensor(ref["pinv"], device="cuda") @ RA).cpu().numpy()
    core_x = None
    qf, rf = O._qr_longdouble(ref["red_l"])
    k = rf.shape[0]; b = qf.T.copy(); x = np.zeros_like(b)
    for i in range(k - 1, -1, -1):
        x[i] = (b[i] - rf[i, i + 1:] @ x[i + 1:]) / rf[i, i]
    core_x = (x @ np.asarray(ref["red_a"], dtype=np.longdouble)).astype(np.float64)
    pinv_x = x.astype(np.float64)
    print(f"== {name}: cond(red_l)={np.linalg.cond(ref['red_l']):.3g}")
    print(f"  pinv: gpu-vs-exact {rel(pinv_g, pinv_x):.2e}  ref-vs-exact {rel(ref['pinv'], pinv_x):.2e}")
    print(f"  core: gpu-vs-exact {rel(core_g, core_x):.2e}  ref-vs-exact {rel(ref['core'], core_x):.2e}"
          f"  solve-vs-exact {rel(core_solve, core_x):.2e}  refpinv@gpu-vs-exact {rel(pinv_cpu_core_gpu, core_x):.2e}")
    print(f"  L: gpu-vs-ref {rel(res.L.numpy(), ref['L']):.2e}  band(ref-vs-exact) {rel(ref['L'], Lx):.2e}"
          f"  gpu-vs-exact {rel(res.L.numpy(), Lx):.2e}")
    print(f"  U: gpu-vs-ref {rel(res.U.numpy(), ref['U']):.2e}  band {rel(ref['U'], Ux):.2e}")
    print(f"  Q equal {np.array_equal(res.Q.indices, ref['Q'])}  P equal {np.array_equal(res.P.indices, ref['P'])}")


if __name__ == "__main__":
    run("smoke", gen_rank_noise(700, 500, 12, 1e-6, 5), dict(r=12, k1=20, l1=80, k2=28, l2=112, seed=7))
    for nm in ("small_dense", "ragged", "tall_f32", "cfg1"):
        a, prm = pipeline_cases()[nm]
        run(nm, a, prm)
