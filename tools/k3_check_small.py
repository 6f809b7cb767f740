"""K3 (apply_sketch_left) vs the oracle at small shapes, K3b v3 and v2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1601_04280_b200 as P
from oracle import draws as D, randlu as O
for (m, n, l, k) in [(300, 18, 104, 26), (300, 240, 104, 26), (2000, 64, 104, 26), (600, 18, 472, 118), (500, 35, 104, 26)]:
    for v2 in (0, 1):
        if v2: os.environ["SRLU_K3B_V2"] = "1"
        else: os.environ.pop("SRLU_K3B_V2", None)
        a = np.random.default_rng(1).standard_normal((m, n))
        om = P.build_composite(k, l, m, "hadamard", 5)
        got = P.apply_sketch_left(om, P.Matrix(a)).numpy()
        ref = O.apply_sketch_left(D.build_composite(k, l, m, 5), a)
        print(m, n, l, k, "v2" if v2 else "v3", "bad", int((got != ref).sum()), "of", got.size)
