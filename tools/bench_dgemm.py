"""Time libsrlu's DMMA GEMM against cuBLAS (torch.mm) on the pipeline's
shapes: core^T = (Omega2 P A)^T pinv^T (n x k2 . k2 x k1) and L = L1 L~
(m x k1 . k1 x k1, lower-triangular B).  CUDA events, median of 20."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_04280_b200.factor import dgemm  # noqa: E402

SHAPES = {  # name: (M, K, N, lower)
    "cfg2_core": (16384, 118, 110, False), "cfg2_L": (16384, 110, 110, True),
    "cfg3_core": (8192, 228, 220, False), "cfg3_L": (262144, 220, 220, True),
    "cfg4_core": (65536, 128, 120, False), "cfg4_L": (1048576, 120, 120, True),
    "cfg5_core": (65536, 558, 550, False), "cfg5_L": (65536, 550, 550, True),
}


def timeit(fn, reps=int(os.environ.get("REPS", "20"))):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    tiles = sys.argv[1:] or [""]
    only = os.environ.get("SHAPES")
    for name, (M, K, N, lower) in SHAPES.items():
        if only and name not in only.split(","):
            continue
        a = torch.randn(M, K, dtype=torch.float64, device="cuda")
        b = torch.randn(K, N, dtype=torch.float64, device="cuda")
        if lower:
            b = torch.tril(b)
        out = torch.empty(M, N, dtype=torch.float64, device="cuda")
        flops = 2.0 * M * N * K
        row = {"shape": name, "M": M, "K": K, "N": N,
               "cublas_ms": timeit(lambda: torch.mm(a, b, out=out))}
        for t in tiles:
            if t:
                os.environ["SRLU_DGEMM_TILE"] = t
            else:
                os.environ.pop("SRLU_DGEMM_TILE", None)
            row[f"srlu{t}_ms"] = timeit(lambda: dgemm(a, b, out=out, b_lower=lower))
        row["cublas_tflops"] = flops / row["cublas_ms"] / 1e9
        for t in tiles:
            row[f"srlu{t}_tflops_dense_equiv"] = flops / row[f"srlu{t}_ms"] / 1e9
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in row.items()}),
              flush=True)


if __name__ == "__main__":
    main()
