import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
g = np.load('tests/golden/pipe_lowrank_resample.npz')
Y = g['Y']; Pref = g['P']
if len(sys.argv) > 1:
    import paper_1601_04280_b200 as P
    r = P.lu_row_pivot(Y)
    print(os.environ.get("SRLU_LU_MAX_GRID"), "equal", np.array_equal(r.P.indices, Pref), r.P.indices[:12], Pref[:12])
    from oracle import randlu as O
    perm, lo, up = O.lu_row_pivot(Y)
    print("L equal", np.array_equal(r.L.numpy(), lo), np.abs(r.L.numpy() - lo).max())
else:
    for cap in ["1", "2", "7", "100", "148"]:
        subprocess.run([sys.executable, __file__, "x"], env=dict(os.environ, SRLU_LU_MAX_GRID=cap))
