"""Golden fixtures for the dense-Gaussian baseline (gaussian_randomized_lu,
reference randlu.py:184-205, 216-219), generated FROM THE REFERENCE ITSELF
in the build container:  python tests/golden/make_golden_gauss.py

The reference's products run on numpy/OpenBLAS (single thread here); the
device runs cuBLAS, so the fixtures pin the permutations and the factors to
within the tolerances of tests/test_gpu_gauss.py, not bit-for-bit."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from tests.golden import cases  # noqa: E402

CASES = {
    "dense": dict(m=300, n=200, r=10, noise=1e-6, seed=11, prm=(10, 3)),
    "tall": dict(m=2000, n=150, r=12, noise=1e-8, seed=12, prm=(12, 5)),
    "sparse": dict(m=400, n=300, r=8, noise=1e-6, seed=13, prm=(8, 7), density=0.3),
}


def main():
    os.environ.setdefault("SPARSELU_BACKEND", "python")
    sys.path.insert(0, "/root/reference/pkg/src")
    from threadpoolctl import threadpool_limits
    import sparselu as sl
    from scipy.sparse import csc_array
    out = {}
    with threadpool_limits(1):
        for name, c in CASES.items():
            a = cases.gen_rank_noise(c["m"], c["n"], c["r"], c["noise"], c["seed"])
            if "density" in c:
                a[np.random.default_rng(c["seed"]).random(a.shape) >= c["density"]] = 0.0
                mat = sl.Matrix(csc_array(a))
            else:
                mat = sl.Matrix(a)
            r, seed = c["prm"]
            prm = sl.default_params(r, c["m"], c["n"], seed=seed)
            res = sl.gaussian_randomized_lu(mat, prm)
            out[name + "_P"] = res.P.indices
            out[name + "_Q"] = res.Q.indices
            out[name + "_L"] = np.asarray(res.L.raw)
            out[name + "_U"] = np.asarray(res.U.raw)
            out[name + "_err"] = np.array(sl.approximation_error(mat, res))
    np.savez_compressed(os.path.join(HERE, "gauss.npz"), **out)
    print("wrote", os.path.join(HERE, "gauss.npz"), sorted(out))


if __name__ == "__main__":
    main()
