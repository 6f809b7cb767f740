"""Benchmark of the B200 sparse randomized LU (BASELINE.json metric:
randomized-LU wall time and GB/s of A streamed vs the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One step = one full ``sparse_randomized_lu`` decomposition of the BASELINE
config's synthetic matrix (default config 2: 16384 x 16384 fp32, k=100,
l=110, width 880; A already resident in HBM).  ``value`` = bytes(A) / step
wall time (GB/s of A per decomposition, whole job); ``e2e`` = the same
through the public API from pinned host memory with the D2H of P, Q, L, U
inside the timed region.  L2 (126 MB) is flushed before every timed step
(and A itself is 1.07 GB > L2).  ``--impl reference`` times the CPU port of
the reference (oracle/, the reference is Python and cannot travel) on the
host cores.  N > 1: one process per GPU under torchrun; A is row-sharded
(paper_1601_04280_b200/dist.py).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs: (m, n, dtype, k, l, width)
CONFIGS = {
    1: dict(m=2048, n=2048, dtype="f64", k=50, l=60, width=480, name="dense 2048x2048 fp64, "
            "sigma_i=exp(-(i-1)/10), Haar U,V"),
    2: dict(m=16384, n=16384, dtype="f32", k=100, l=110, width=880, name="dense 16384x16384 fp32, "
            "sigma_i=i^-2, Haar U,V, + N(0,1e-6) noise (std)"),
    3: dict(m=262144, n=8192, dtype="f32", k=200, l=220, width=1760, name="tall dense 262144x8192 "
            "fp32, G1 G2 + N(0,1e-3) noise (std)"),
    4: dict(m=1048576, n=65536, dtype="csr-f32", k=100, l=120, width=960, name="CSR 1048576x65536 "
            "fp32, 0.1% i.i.d. positions, N(0,1) values"),
    5: dict(m=65536, n=65536, dtype="f64", k=500, l=550, width=4400, name="dense 65536x65536 fp64, "
            "Haar rank 1000, sigma_i=10^(-4(i-1)/999), + N(0,1e-8) noise (std)"),
}
HAAR_RANK_CFG2 = 16384  # full 16384 x 16384 Haar factors, as BASELINE config 2 states


def _gen(seed, device):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _haar_cols(m, r, g, device):
    x = torch.randn(m, r, generator=g, device=device, dtype=torch.float64)
    q, rr = torch.linalg.qr(x)
    return q * torch.sign(torch.diagonal(rr))


GEN_BLOCK = 4096   # rows per independently seeded block of the generators


def _blocks(r0, r1):
    return range(r0 // GEN_BLOCK, (r1 + GEN_BLOCK - 1) // GEN_BLOCK)


def _block_noise(c, b, n, std, device, dtype):
    """Noise of generator block b (rows [b*GEN_BLOCK, (b+1)*GEN_BLOCK)):
    its own seed, so any row range is generated identically alone or as
    part of the whole matrix (row-sharded ranks generate only their rows)."""
    g = _gen((1000 + c) * 1000003 + b, device)
    return std * torch.randn(GEN_BLOCK, n, generator=g, device=device, dtype=dtype)


def gen_config(c, device="cuda", row_range=None):
    """Synthetic A of BASELINE config c on the device (deterministic per
    seed) and its RandLuParams fields; ``row_range=(r0, r1)`` generates only
    those rows (the same values as the full matrix's rows: the noise and the
    row factors are seeded per 4096-row block).  Noise 'N(0,v)' is read as
    standard deviation v."""
    from paper_1601_04280_b200 import params_from_north_star
    cfg = CONFIGS[c]
    m, n = cfg["m"], cfg["n"]
    r0, r1 = row_range if row_range is not None else (0, m)
    prm = params_from_north_star(m, n, cfg["k"], cfg["l"], cfg["width"], seed=0)
    prm = dict(r=prm.r, k1=prm.k1, l1=prm.l1, k2=prm.k2, l2=prm.l2, seed=0)
    g = _gen(1000 + c, device)

    def rows_of(fn, dtype):
        out = []
        for b in _blocks(r0, r1):
            blk = fn(b)
            lo, hi = max(r0, b * GEN_BLOCK), min(r1, (b + 1) * GEN_BLOCK)
            out.append(blk[lo - b * GEN_BLOCK:hi - b * GEN_BLOCK].to(dtype))
        return torch.cat(out, 0).contiguous()

    if c == 1:
        from tests.golden.cases import config1_matrix
        from threadpoolctl import threadpool_limits
        with threadpool_limits(1):
            a = torch.from_numpy(config1_matrix()).to(device)
        return a[r0:r1].contiguous(), prm
    if c in (2, 5):
        # U, V: Haar of rank r (QR of seeded N(0,1) with the sign fix), whole
        # on every rank (m x r); A rows = U[rows] diag(sigma) V^T + noise
        r = min(HAAR_RANK_CFG2, m, n) if c == 2 else 1000
        u = _haar_cols(m, r, g, device)
        v = _haar_cols(n, r, g, device)
        if c == 2:
            s = torch.arange(1, r + 1, device=device, dtype=torch.float64) ** -2.0
            std, dt = 1e-6, torch.float32
        else:
            s = 10.0 ** (-4.0 * torch.arange(r, device=device, dtype=torch.float64) / 999.0)
            std, dt = 1e-8, torch.float64
        us = u * s
        del u

        def blk(b):
            lo = b * GEN_BLOCK
            x = us[lo:lo + GEN_BLOCK] @ v.t()
            nz = _block_noise(c, b, n, std, device, torch.float64)
            x += nz[:x.shape[0]]
            return x

        return rows_of(blk, dt), prm
    if c == 3:
        g2 = torch.randn(200, n, generator=g, device=device) / math.sqrt(200.0)

        def blk(b):
            gb = _gen((1000 + c) * 1000003 + b, device)
            g1 = torch.randn(GEN_BLOCK, 200, generator=gb, device=device) / math.sqrt(200.0)
            x = g1 @ g2
            x += 1e-3 * torch.randn(GEN_BLOCK, n, generator=gb, device=device)
            return x

        return rows_of(blk, torch.float32), prm
    if c == 4:
        # per 4096-row block: round(4096 n 1e-3) i.i.d. uniform positions in
        # the block (stratified i.i.d.), values N(0,1), duplicates summed
        nnz_b = int(round(GEN_BLOCK * n * 1e-3))
        ptrs, idxs, vals = [torch.zeros(1, dtype=torch.int64, device=device)], [], []
        base = 0
        for b in _blocks(r0, r1):
            gb = _gen((1000 + c) * 1000003 + b, device)
            rows = torch.randint(0, GEN_BLOCK, (nnz_b,), generator=gb, device=device)
            cols = torch.randint(0, n, (nnz_b,), generator=gb, device=device)
            vv = torch.randn(nnz_b, generator=gb, device=device, dtype=torch.float64)
            lo, hi = max(r0, b * GEN_BLOCK), min(r1, (b + 1) * GEN_BLOCK)
            keep = (rows >= lo - b * GEN_BLOCK) & (rows < hi - b * GEN_BLOCK)
            rows, cols, vv = rows[keep] - (lo - b * GEN_BLOCK), cols[keep], vv[keep]
            key = rows * n + cols
            key, order = torch.sort(key)
            vv = vv[order]
            uk, inv = torch.unique_consecutive(key, return_inverse=True)
            sv = torch.zeros(uk.numel(), dtype=torch.float64, device=device).index_add_(0, inv, vv)
            rr = uk // n
            cnt = torch.bincount(rr, minlength=hi - lo)
            ptrs.append(base + torch.cumsum(cnt, 0))
            base += int(uk.numel())
            idxs.append((uk % n).to(torch.int32))
            vals.append(sv.float())
        return (torch.cat(ptrs), torch.cat(idxs), torch.cat(vals)), prm
    raise ValueError(c)


def a_bytes(a):
    if isinstance(a, tuple):
        return sum(t.numel() * t.element_size() for t in a)
    return a.numel() * a.element_size()


def as_matrix(P, a, shape):
    if isinstance(a, tuple):
        return P.Matrix.from_csr(*a, shape=shape)
    return P.Matrix.from_device(a)


# --------------------------------------------------------------------------
# measurement helpers


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during a region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device_index=0, interval=0.005):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._h = None
        self.interval = interval

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                break
            time.sleep(self.interval)

    def __enter__(self):
        if self._h is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._h is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml-unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


_flush_buf = None


def flush_l2():
    global _flush_buf
    if _flush_buf is None:
        _flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    _flush_buf.fill_(1)


def time_region(fn, steps, flush=True, barrier=None, kernel=False):
    """Per-step CUDA-event times (ms) on the current stream; L2 flushed
    before every step outside the timed span.  kernel=True (single-kernel
    timings for the rooflines): the start event is enqueued behind the L2
    flush without a host sync, so the host's launch latency overlaps the
    flush instead of being counted as kernel time."""
    times = []
    for _ in range(steps):
        if flush:
            flush_l2()
        if not kernel:
            torch.cuda.synchronize()
        if barrier:
            barrier()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e))
    return times


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config):
    """dram read+write bytes per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(str(config), {}).get("k1_dram_bytes")


# --------------------------------------------------------------------------
# CPU legs (oracle port of the reference)


def cpu_reference(a_host, prm, steps, threads):
    from threadpoolctl import threadpool_limits
    from oracle import randlu as O
    times = []
    with threadpool_limits(threads):
        for _ in range(steps):
            t = time.perf_counter()
            O.sparse_randomized_lu(a_host, prm)
            times.append(time.perf_counter() - t)
    return times


def host_copy(a, shape):
    if isinstance(a, tuple):
        from scipy.sparse import csr_array
        indptr, indices, vals = (t.cpu().numpy() for t in a)
        return csr_array((vals.astype(np.float64), indices, indptr), shape=shape)
    return a.double().cpu().numpy()


# --------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--dist", action="store_true",
                    help="use the row-sharded path even at world size 1 (NCCL)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    metric = "randomized-LU GB/s of A streamed per decomposition (wall time of sparse_randomized_lu)"
    workload = f"BASELINE config {args.config}: {cfg['name']}, k={cfg['k']}, l={cfg['l']}, " \
               f"CountSketch width {cfg['width']}"

    if args.impl == "reference":
        if rank != 0:
            return
        return run_reference_arm(args, cfg, metric, workload)

    torch.cuda.set_device(local)
    if world > 1 or args.dist:
        import torch.distributed as dist
        if "MASTER_ADDR" not in os.environ:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0",
                              WORLD_SIZE="1", LOCAL_RANK="0")
        dist.init_process_group("nccl")
        from paper_1601_04280_b200 import dist as D
        return D.bench_main(args, cfg, metric, workload, gen_config, time_region, flush_l2,
                            ClockSampler, measured_peaks)

    import paper_1601_04280_b200 as P
    from paper_1601_04280_b200 import _lib
    from paper_1601_04280_b200.sketch import sketch_right_into, sketch_left_into, members

    a, prm_d = gen_config(args.config)
    shape = (cfg["m"], cfg["n"])
    A = as_matrix(P, a, shape)
    params = P.RandLuParams(**prm_d)
    nbytes = a_bytes(a)
    torch.cuda.synchronize()

    step = lambda: P.sparse_randomized_lu(A, params)
    for _ in range(max(3, args.warmup)):
        res = step()
    _lib.LAUNCHES.reset()
    with ClockSampler(local) as clk:
        times = time_region(step, args.steps)
    launches = _lib.LAUNCHES.total
    ms = float(np.mean(times))
    value = nbytes / (ms / 1e3) / 1e9
    res = step()
    stages = {k: round(v * 1e3, 4) for k, v in res.elapsed.items()}

    # ---- dominant streaming kernel (K1: fused sketch of A) live ----------
    om1 = res.extras.get("omega1") if res.extras else None
    ops = P.randlu._CompositeOps(params, shape[0], shape[1], 0, 1, A.device)
    y = torch.empty(shape[0], params.k1, dtype=torch.float64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    ops.omega1.sem.plan()
    sketch_right_into(A, ops.omega1, y, flag)  # builds the K1 gather schedule (once per sketch)
    k1_sched = any(v is not None for _, v in ops.omega1.sem._sched)
    k1_times = time_region(lambda: sketch_right_into(A, ops.omega1, y, flag), args.steps,
                           kernel=True)
    k1_ms = float(np.mean(k1_times))
    k1_bytes = nbytes + y.numel() * 8
    # K3 (projection stream of P A)
    perm = torch.randperm(shape[0], device="cuda")
    out = torch.empty(shape[1], params.k2, dtype=torch.float64, device="cuda")
    if A.is_sparse:
        inv = torch.empty(shape[0], dtype=torch.int32, device="cuda")
        inv[perm] = torch.arange(shape[0], dtype=torch.int32, device="cuda")
        k3 = lambda: sketch_left_into(A, ops.omega2, None, None, None, out, inv_perm=inv,
                                      flags=flag)
    else:
        mrow, msign, bptr = members(ops.omega2, perm, 0, shape[0])
        k3 = lambda: sketch_left_into(A, ops.omega2, mrow, msign, bptr, out)
    k3_ms = float(np.mean(time_region(k3, args.steps, kernel=True)))
    k3_bytes = nbytes + out.numel() * 8
    peak, peak_src = measured_peaks()
    k1_gbs = k1_bytes / (k1_ms / 1e3) / 1e9
    k3_gbs = k3_bytes / (k3_ms / 1e3) / 1e9
    traffic = ncu_traffic(args.config)

    # ---- e2e through the public API from pinned host memory ------------
    e2e_steps = args.e2e_steps or min(args.steps, 5)
    if isinstance(a, tuple):
        host_a = tuple(t.cpu().pin_memory() for t in a)
    else:
        host_a = a.cpu().pin_memory()
    d2h = {}

    def e2e_step():
        if isinstance(host_a, tuple):
            dev = tuple(t.to("cuda", non_blocking=True) for t in host_a)
            mat = P.Matrix.from_csr(*dev, shape=shape)
        else:
            mat = P.Matrix.from_device(host_a.to("cuda", non_blocking=True))
        r = P.sparse_randomized_lu(mat, params)
        lh = r.L.to_host()  # pinned D2H through the public Matrix API
        uh = r.U.to_host()
        d2h["bytes"] = lh.numel() * 8 + uh.numel() * 8 + r.P.size * 8 + r.Q.size * 8

    e2e_step()
    e2e_times = time_region(e2e_step, e2e_steps)
    e2e_ms = float(np.mean(e2e_times))

    line = {
        "metric": metric, "value": round(value, 3), "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4),
        "step_ms": {"min": round(float(np.min(times)), 4), "median": round(float(np.median(times)), 4),
                    "max": round(float(np.max(times)), 4)},
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, generated on device; BASELINE config shapes)",
        "config": {"workload": workload, "config_id": args.config, "m": shape[0], "n": shape[1],
                   "a_dtype": cfg["dtype"], "bytes_A": nbytes, "params": prm_d,
                   "l2": "flushed before every timed step (256 MiB write); A > L2",
                   "parallelism": "single GPU"},
        "stages_ms": stages,
        "roofline": {"bound": "hbm", "kernel": ("k1s_kernel (scheduled, warp-specialised fused CountSketch+FWHT "
                                "sketch of A, stage 1)" if k1_sched else
                                "k1v2_kernel (fused CountSketch+FWHT sketch of A, stage 1)")
                     if not A.is_sparse else "k1_csr_kernel",
                     "achieved": round(k1_gbs, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(k1_gbs / peak, 4), "traffic": traffic,
                     "algorithmic_bytes": k1_bytes, "avg_launch_ms": round(k1_ms, 4),
                     "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)"},
        "kernels": {"k3_sketch_left": {"avg_launch_ms": round(k3_ms, 4),
                                       "achieved_gbs": round(k3_gbs, 1),
                                       "frac": round(k3_gbs / peak, 4),
                                       "algorithmic_bytes": k3_bytes}},
        "e2e": {"value": round(nbytes / (e2e_ms / 1e3) / 1e9, 3), "unit": "GB/s",
                "ms_per_step": round(e2e_ms, 3), "steps": e2e_steps,
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": d2h.get("bytes")},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(a, shape, prm_d, nbytes)
    print(json.dumps(line), flush=True)


def cpu_baseline(a, shape, prm, nbytes, steps=1):
    threads = os.cpu_count() or 1
    host = host_copy(a, shape)
    times = cpu_reference(host, prm, steps, threads)
    t = float(np.mean(times))
    return {"value": round(nbytes / t / 1e9, 5), "unit": "GB/s", "cores": threads,
            "kind": "port", "seconds_per_decomposition": round(t, 3),
            "sample": f"{steps} full decomposition(s) of the same A by the oracle/ CPU port of "
                      f"the reference (numpy+C, BLAS threads={threads})"}


def run_reference_arm(args, cfg, metric, workload):
    steps = max(1, min(args.steps, 3))
    warm = min(args.warmup, 1)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    a, prm = gen_config(args.config, dev)
    shape = (cfg["m"], cfg["n"])
    nbytes = a_bytes(a)
    host = host_copy(a, shape)
    del a
    threads = os.cpu_count() or 1
    if warm:
        cpu_reference(host, prm, warm, threads)
    times = cpu_reference(host, prm, steps, threads)
    t = float(np.mean(times))
    v = nbytes / t / 1e9
    line = {
        "impl": "reference", "metric": metric, "value": round(v, 5), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": round(t * 1e3, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (same generator and seed as the GPU arm)",
        "config": {"workload": workload, "config_id": args.config, "m": shape[0],
                   "n": shape[1], "bytes_A": nbytes, "params": prm},
        "cpu_baseline": {"value": round(v, 5), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{steps} full decomposition(s) (steps capped at 3 to bound "
                                   f"the CPU run) by the oracle/ port of the reference"},
        "e2e": {"value": round(v, 5), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
