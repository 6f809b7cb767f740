"""K1T probe: Y bit-exact vs the oracle for a forced rows-per-block (SRLU_K1T_ROWS)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_04280_b200 as P
from oracle import draws as D
from oracle import randlu as O

m, n, l, k = [int(x) for x in sys.argv[1:5]]
dt = np.float32 if (len(sys.argv) < 6 or sys.argv[5] == "f32") else np.float64
rng = np.random.default_rng(5)
a = (rng.standard_normal((m, n)) * 10.0 ** rng.integers(-20, 20, size=(m, n))).astype(dt)
om = P.build_composite(k, l, n, "hadamard", 7)
y = P.apply_sketch_right(P.Matrix.from_device(torch.from_numpy(a).cuda()), om).numpy()
ref = O.apply_sketch_right(a.astype(np.float64), D.build_composite(k, l, n, 7))
bad = np.argwhere(y != ref)
print("rows", os.environ.get("SRLU_K1T_ROWS"), "shape", (m, n, l, k), dt.__name__,
      "OK" if bad.size == 0 else f"MISMATCH {len(bad)} first {bad[:5].tolist()} rows {sorted(set(bad[:,0].tolist()))[:40]}")
