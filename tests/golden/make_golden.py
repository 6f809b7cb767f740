"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--ref-src /tmp/refbuild/src]

It imports the reference package ``sparselu`` (arxiv/paper_1601_04280,
/root/reference/pkg/src/sparselu) — preferably a scratch build with the
compiled Cython lane (``cp -r /root/reference/pkg /tmp/refbuild && cd
/tmp/refbuild && python setup.py build_ext --inplace``), otherwise the
read-only source tree with ``SPARSELU_BACKEND=python`` (the reference
tests the two lanes bitwise equal, tests/test_kernels.py:111-136) — runs it
on small seeded inputs and freezes its outputs as .npz files.  Nothing
here runs on the GPU box; the fixtures travel instead.

Inputs are regenerated deterministically by tests/golden/cases.py, so
only outputs (plus a sha256 of each input) are stored.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests.golden import cases  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def import_reference(ref_src):
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    if ref_src is None:
        if os.path.exists("/tmp/refbuild/src/sparselu/_kernels"):
            ref_src = "/tmp/refbuild/src"
        else:
            ref_src = "/root/reference/pkg/src"
            os.environ["SPARSELU_BACKEND"] = "python"
    sys.path.insert(0, ref_src)
    import sparselu  # noqa: F401
    return sparselu


def pipeline_with_intermediates(sl, a, params):
    """Re-run the reference's _attempt (randlu.py:246-276) with its own
    functions, keeping the intermediates; asserts the final factors equal
    sparse_randomized_lu's."""
    from sparselu import randlu as R
    from sparselu.matrix import permute_rows, matmul
    from sparselu.factor import lu_row_pivot, lu_col_pivot, left_pseudo_inverse
    res = sl.sparse_randomized_lu(a, params)
    m, n = a.shape
    attempt = None
    for t in range(1 + R.MAX_RESAMPLES):
        ops = R._CompositeOps(params, m, n, params.seed + 2 * t, params.seed + 2 * t + 1)
        y = ops.project_right(a)
        first = lu_row_pivot(y)
        red_l = ops.project_left(first.L)
        red_a = ops.project_left(permute_rows(first.P, a))
        try:
            pinv = left_pseudo_inverse(red_l)
        except sl.SingularMatrixError:
            continue
        attempt = t
        break
    core = matmul(pinv, red_a)
    second = lu_col_pivot(core)
    lf = matmul(first.L, second.L)
    assert np.array_equal(res.P.indices, first.P.indices)
    assert np.array_equal(res.Q.indices, second.Q.indices)
    assert np.array_equal(res.L.to_dense(), lf.to_dense())
    assert np.array_equal(res.U.to_dense(), second.U.to_dense())
    err = sl.approximation_error(a, res)
    return dict(
        attempt=np.int64(attempt),
        Y=y.to_dense(), P=res.P.indices, L1=first.L.to_dense(),
        red_l=red_l.to_dense(), red_a=red_a.to_dense(), pinv=pinv.to_dense(),
        core=core.to_dense(), Q=res.Q.indices, Lt=second.L.to_dense(),
        L=res.L.to_dense(), U=res.U.to_dense(), err=np.float64(err),
        om1_row_of=ops.omega1.sem.row_of, om1_sign=ops.omega1.sem.sign,
        om1_phase=ops.omega1.fast.phase, om1_idx=ops.omega1.fast.sample_idx,
        om2_row_of=ops.omega2.sem.row_of, om2_sign=ops.omega2.sem.sign,
        om2_phase=ops.omega2.fast.phase, om2_idx=ops.omega2.fast.sample_idx,
    )


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref-src", default=None)
    args = ap.parse_args()
    sl = import_reference(args.ref_src)
    print("reference lane:", sl.KERNEL_BACKEND)
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        # ---- kernels (the plugin seam, _kernels/__init__.py) -------------
        from sparselu import _kernels as K
        kern = {}
        for name, case in cases.kernel_cases().items():
            kind = case["kind"]
            if kind == "fwht":
                x = case["x"].copy()
                K.fwht_rows(x)
                kern[name] = x
            elif kind in ("gather_dense", "scatter_dense"):
                a = np.asfortranarray(case["a"])
                out = np.zeros(case["out_shape"], order="F")
                getattr(K, "sem_" + kind)(a, case["row_of"], case["sign"], out)
                kern[name] = out
            else:
                sp = case["csc"]
                out = np.zeros(case["out_shape"], order="F")
                getattr(K, "sem_" + kind)(sp.data, sp.indices, sp.indptr,
                                          case["row_of"], case["sign"], out)
                kern[name] = out
        np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kern)

        # ---- draws at every BASELINE config shape ------------------------
        dr = {}
        for name, (k, l, n, seed) in cases.DRAW_SHAPES.items():
            om = sl.build_composite(k, l, n, "hadamard", seed)
            dr[name + "_row_of_sha"] = np.bytes_(sha(om.sem.row_of.astype(np.int64)))
            dr[name + "_sign_sha"] = np.bytes_(sha(om.sem.sign.astype(np.float64)))
            dr[name + "_row_of_head"] = om.sem.row_of[:64]
            dr[name + "_sign_head"] = om.sem.sign[:64]
            dr[name + "_phase"] = om.fast.phase
            dr[name + "_idx"] = om.fast.sample_idx
            dr[name + "_pad"] = np.int64(om.fast.pad)
            dr[name + "_scale"] = np.float64(om.fast.scale)
        np.savez_compressed(os.path.join(HERE, "draws.npz"), **dr)

        # ---- factorizations (factor.py) ----------------------------------
        fac = {}
        for name, b in cases.factor_cases().items():
            r = sl.lu_row_pivot(sl.Matrix(b)) if b.shape[0] >= b.shape[1] else None
            if r is not None:
                fac[name + "_row_P"] = r.P.indices
                fac[name + "_row_L"] = r.L.to_dense()
                fac[name + "_row_U"] = r.U.to_dense()
            bt = b.T if b.shape[0] >= b.shape[1] else b
            c = sl.lu_col_pivot(sl.Matrix(bt))
            fac[name + "_col_Q"] = c.Q.indices
            fac[name + "_col_L"] = c.L.to_dense()
            fac[name + "_col_U"] = c.U.to_dense()
        np.savez_compressed(os.path.join(HERE, "factor.npz"), **fac)

        # ---- full pipeline ------------------------------------------------
        for name, (a, prm) in cases.pipeline_cases().items():
            params = sl.RandLuParams(**prm)
            mat = sl.Matrix(a) if not hasattr(a, "tocsc") else sl.Matrix.sparse(a)
            out = pipeline_with_intermediates(sl, mat, params)
            dense_in = a.toarray() if hasattr(a, "toarray") else a
            out["a_sha"] = np.bytes_(sha(np.asarray(dense_in, dtype=np.float64)))
            if a.shape[0] > 1000:  # keep the big fixtures lean
                for key in ("L1", "pinv", "Lt"):
                    out.pop(key)
            np.savez_compressed(os.path.join(HERE, f"pipe_{name}.npz"), **out)
            print(name, a.shape, "attempt", int(out["attempt"]), "err", float(out["err"]))


if __name__ == "__main__":
    main()
