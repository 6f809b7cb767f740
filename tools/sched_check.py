"""K1 schedule determinism check: build the schedule for a config's shape
and print a hash of its codes (compare across builds/variants)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
if len(sys.argv) > 1:
    import paper_1601_04280_b200._lib as _L
    _L.LIB_PATH = sys.argv[1]
import paper_1601_04280_b200 as P
for (k, l, n, dt) in [(110, 880, 16384, 0), (220, 1760, 8192, 0), (60, 480, 2048, 1), (100, 3000, 30000, 0)]:
    om = P.build_composite(k, l, n, "hadamard", 0)
    s = om.sem.k1_schedule(dt, om.fast.pad)
    torch.cuda.synchronize()
    words = int(s[:4].view(torch.int32)[0].item())
    print(n, l, "code words", words, flush=True)
