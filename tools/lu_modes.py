"""Run lu_row_pivot / lu_col_pivot once on a random (m x k) input under the
current SRLU_LU_* env and compare with the oracle.  Usage:
  python tools/lu_modes.py row|col m k"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1601_04280_b200 as P
from oracle import randlu as O

mode, m, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
g = np.random.Generator(np.random.Philox(m + k))
b = g.standard_normal((m, k))
if mode == "row":
    r = P.lu_row_pivot(b)
    perm, lo, up = O.lu_row_pivot(b)
    ok = np.array_equal(r.P.indices, perm) and np.array_equal(r.L.numpy(), lo) and np.array_equal(r.U.numpy(), up)
else:
    c = b.T.copy()
    r = P.lu_col_pivot(c)
    q, lo, up = O.lu_col_pivot(c)
    ok = np.array_equal(r.Q.indices, q) and np.array_equal(r.L.numpy(), lo) and np.array_equal(r.U.numpy(), up)
print(mode, m, k, {k_: v for k_, v in os.environ.items() if k_.startswith("SRLU_LU")}, "exact" if ok else "DIFFERS")
