"""Host->device bandwidth from pinned memory: one copy vs the same bytes
split over several streams (copy engines) — informs the e2e upload path."""
import sys, time
import torch
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for nstreams in (1, 2, 4, 8):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ch = n // nstreams
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * ch:(i + 1) * ch].copy_(h[i * ch:(i + 1) * ch], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"{nstreams} streams: {n / dt / 1e9:.1f} GB/s", flush=True)
# D2H
torch.cuda.synchronize(); t = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize()
print(f"D2H 1 stream: {n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max", "--format=csv"], capture_output=True, text=True).stdout)
