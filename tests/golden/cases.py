"""Deterministic inputs shared by the golden generator (which runs the
reference on them) and by the parity tests (which run the oracle and the
CUDA path on them).  Everything is derived from numpy Philox seeds with
single-threaded numpy, so the same bits come out in the build container
and on the GPU box (same image)."""

from __future__ import annotations

import numpy as np
from scipy.sparse import csc_array, random_array


def _g(seed):
    return np.random.Generator(np.random.Philox(seed))


def kernel_cases():
    c = {}
    for n in (1, 2, 4, 16, 64, 256, 1024):
        c[f"fwht_{n}"] = dict(kind="fwht", x=_g(100 + n).standard_normal((6, n)))
    for name, (m, n, l, seed) in dict(gd1=(13, 21, 6, 10), gd2=(31, 47, 9, 14)).items():
        g = _g(seed)
        c[name] = dict(kind="gather_dense", a=g.standard_normal((m, n)),
                       row_of=g.integers(0, l, size=n),
                       sign=(g.integers(0, 2, size=n) * 2 - 1).astype(np.float64),
                       out_shape=(m, l))
    for name, (m, n, l, seed) in dict(sd1=(19, 8, 5, 12), sd2=(64, 33, 7, 15)).items():
        g = _g(seed)
        c[name] = dict(kind="scatter_dense", a=g.standard_normal((m, n)),
                       row_of=g.integers(0, l, size=m),
                       sign=(g.integers(0, 2, size=m) * 2 - 1).astype(np.float64),
                       out_shape=(l, n))
    for name, (m, n, l, seed, kind) in dict(
            gc1=(17, 29, 7, 11, "gather_csc"), sc1=(23, 11, 4, 13, "scatter_csc"),
            gc2=(40, 90, 12, 16, "gather_csc")).items():
        g = _g(seed)
        d = g.standard_normal((m, n))
        d[g.random((m, n)) < 0.6] = 0
        sp = csc_array(d)
        sp.indices = sp.indices.astype(np.int64)
        sp.indptr = sp.indptr.astype(np.int64)
        cnt = n if kind == "gather_csc" else m
        c[name] = dict(kind=kind, csc=sp, dense=d,
                       row_of=g.integers(0, l, size=cnt),
                       sign=(g.integers(0, 2, size=cnt) * 2 - 1).astype(np.float64),
                       out_shape=(m, l) if kind == "gather_csc" else (l, n))
    return c


# (k, l, in_dim, seed) of build_composite at every BASELINE config shape
# (omega1 uses seed, omega2 seed+1) plus odd shapes
DRAW_SHAPES = {
    "c1_om1": (60, 480, 2048, 0), "c1_om2": (68, 272, 2048, 1),
    "c2_om1": (110, 880, 16384, 0), "c2_om2": (118, 472, 16384, 1),
    "c3_om1": (220, 1760, 8192, 0), "c3_om2": (228, 912, 262144, 1),
    "c4_om1": (120, 960, 65536, 0), "c4_om2": (128, 512, 1048576, 1),
    "c5_om1": (550, 4400, 65536, 0), "c5_om2": (558, 2232, 65536, 1),
    "odd1": (3, 12, 16, 7), "odd2": (5, 9, 15, 2 ** 33 + 5),
    "odd3": (1, 2, 2, 12345), "odd4": (17, 17, 17, 3),
}


def factor_cases():
    c = {}
    g = _g(0)
    c["rand_40x12"] = g.standard_normal((40, 12))
    c["rand_200x30"] = _g(1).standard_normal((200, 30))
    # small integers: many exact ties in |w| -> first-index tie breaking
    c["ties_60x9"] = _g(2).integers(-2, 3, size=(60, 9)).astype(np.float64)
    c["ties_16x16"] = _g(3).integers(-1, 2, size=(16, 16)).astype(np.float64)
    c["zero_5x3"] = np.zeros((5, 3))
    g4 = _g(4)
    c["lowrank_30x10"] = g4.standard_normal((30, 4)) @ g4.standard_normal((4, 10))
    c["eye_3"] = np.eye(3)
    c["swap_2"] = np.array([[0.0, 1.0], [1.0, 0.0]])
    c["hand_col"] = np.array([[1.0, 5.0], [0.0, 1.0]]).T  # col-pivot hand case
    c["tiny_1x1"] = np.array([[-3.0]])
    c["col_ones"] = np.ones((7, 3))
    return c


def gen_rank_noise(m, n, r, noise, seed):
    g = _g(seed)
    return g.standard_normal((m, r)) @ g.standard_normal((r, n)) + noise * g.standard_normal((m, n))


def haar(g, m, r):
    """First r columns of a Haar-orthonormal m x m matrix (QR of N(0,1),
    sign fix so diag(R) > 0)."""
    q, rr = np.linalg.qr(g.standard_normal((m, r)))
    return q * np.sign(np.diag(rr))


def config1_matrix():
    """BASELINE config 1: 2048^2 fp64, A = U diag(exp(-(i-1)/10)) V^T."""
    g = _g(1)
    n = 2048
    u = haar(g, n, n)
    v = haar(g, n, n)
    s = np.exp(-np.arange(n) / 10.0)
    return (u * s) @ v.T


# seed for which the reference's first attempt hits a rank-deficient
# reduced system and resamples (found by scanning with the reference)
RESAMPLE_SEED = 37


def pipeline_cases():
    c = {}
    c["small_dense"] = (gen_rank_noise(300, 240, 10, 1e-6, 7),
                        dict(r=10, k1=18, l1=72, k2=26, l2=104, seed=3))
    c["ragged"] = (_g(8).standard_normal((257, 131)),
                   dict(r=5, k1=9, l1=37, k2=15, l2=61, seed=11))
    g = _g(9)
    d = g.standard_normal((400, 300))
    d[g.random((400, 300)) < 0.97] = 0.0
    c["sparse"] = (csc_array(d), dict(r=6, k1=14, l1=56, k2=22, l2=88, seed=5))
    c["zero"] = (np.zeros((60, 50)), dict(r=2, k1=3, l1=20, k2=4, l2=48, seed=1))
    c["lowrank_resample"] = (gen_rank_noise(100, 90, 5, 0.0, 21),
                             dict(r=5, k1=13, l1=52, k2=21, l2=84, seed=RESAMPLE_SEED))
    t = gen_rank_noise(2000, 300, 20, 1e-3, 10).astype(np.float32).astype(np.float64)
    c["tall_f32"] = (t, dict(r=20, k1=30, l1=120, k2=38, l2=152, seed=0))
    g = _g(11)
    sp = random_array((5000, 1200), density=0.005, format="csr", rng=g,
                      data_sampler=g.standard_normal).astype(np.float32).astype(np.float64)
    c["sparse_wide"] = (csc_array(sp), dict(r=10, k1=18, l1=72, k2=26, l2=104, seed=2))
    c["cfg1"] = (config1_matrix(), dict(r=50, k1=60, l1=480, k2=68, l2=272, seed=0))
    return c
