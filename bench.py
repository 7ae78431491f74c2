#!/usr/bin/env python
"""Benchmark of the conv-as-SpMV hot path (BASELINE.json metric).

Workload (default, --config 3): BASELINE config 3 -- a global batch of 256
1024x1024 fp32 images, 3x3 kernel, s=1, p=1, applied as a batched SpMM of the
CSR transform T (9,424,900 stored entries).  With N GPUs (torchrun, one rank
per GPU) every rank builds its own CSR replica on its device and owns a
contiguous slice of the batch; there is no collective on the data path.

One step = one spconv_spmm call over this rank's images (the CSR band check
+ the register-blocked apply: two launches), inputs resident in HBM (config
3's 1 GB X slice is larger than the 126 MB L2, so no flush is needed; working
sets under 2x L2 get a 512 MB scrub write + a 512 MB read between steps, outside the
timed events, so L2 is cold and clean).
Scaling is weak: each rank owns per_gpu_batch images.  value = whole-job
nnz-MACs per second (total images x nnz / max-over-ranks device time).
e2e = the same metric through the C ABI with pinned HOST buffers (H2D + SpMM
+ D2H pipelined in the library).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# per_gpu_batch: images each rank owns (weak scaling: the job grows with N).
CONFIGS = {
    1: dict(spec=(64, 64, 3, 1, 1), per_gpu_batch=1, name="config1: 64x64 single image, k3 s1 p1"),
    2: dict(spec=(512, 512, 5, 2, 2), per_gpu_batch=1,
            name="config2: 512x512 single image, k5 s2 p2 SpMV"),
    3: dict(spec=(1024, 1024, 3, 1, 1), per_gpu_batch=256,
            name="config3: 1024x1024 images, k3 s1 p1, batched SpMM, 256 images per GPU"),
    4: dict(spec=(4096, 4096, 7, 2, 3), per_gpu_batch=8,
            name="config4: 4096x4096 images, k7 s2 p3, build + batched SpMM, 8 images per GPU "
                 "(batch 64 over 8 GPUs)"),
}
METRIC = "SpMV-conv nnz-MAC/s (whole job) with HBM GB/s and CSR build ms"
UNIT = "G nnz-MAC/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(cfg: int, batch: int):
    """DRAM bytes (read + write) of one spmm call at this config and per-GPU
    batch, from the newest committed ncu --set full capture (profiles/*/
    ncu_summary.json, written by scripts/make_profiles.py); None if absent."""
    import glob
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_summary.json")), reverse=True)
    latest = os.path.join(ROOT, "profiles", "LATEST")  # tag of the newest evidence pass (make_profiles.py)
    if os.path.exists(latest):
        with open(latest) as f:
            first = os.path.join(ROOT, "profiles", f.read().strip(), "ncu_summary.json")
        paths = [first] + [q for q in paths if q != first]
    for path in paths:
        try:
            with open(path) as f:
                j = json.load(f)
        except Exception:
            continue
        hits = [e for e in j.values() if e.get("config") == cfg and e.get("batch") == batch
                and e.get("role") == "spmm"]
        if hits:
            return sum(e["dram_bytes_per_launch"] for e in hits), ", ".join(e["source"] for e in hits)
    return None, None


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML every `period` s."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, device_index: int, period: float = 0.005):
        self.samples = []  # (t, sm_mhz, reasons_mask)
        self.period = period
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, int(rs)))
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._t.start()
        return self

    def stop(self):
        self._stop.set()
        if self.ok:
            self._t.join(1.0)

    def summary(self, t0: float, t1: float):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        busy = [s for s in win if not (s[2] & 0x1)] or win or self.samples
        mask = 0
        for s in busy:
            mask |= s[2]
        reasons = sorted(k for k, v in self.REASONS.items() if mask & v and k != "gpu_idle")
        return {"sm_mhz": statistics.median(s[1] for s in busy), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(busy)}


def algorithmic_bytes(rows, cols, nnz, b):
    """8*nnz + 4*(rows+1) + 4*b*(cols+rows) per launch (matrix read once)."""
    return 8 * nnz + 4 * (rows + 1) + 4 * b * (cols + rows)


# ----------------------------------------------------------------------------
# CPU baseline: the reference's own convolve() (oracle/_ref) on a bounded sample
# ----------------------------------------------------------------------------

def cpu_baseline(spec, seconds: float = 10.0):
    import oracle
    m, n, k, s, p = spec
    cores = os.cpu_count() or 1
    ref = oracle.try_ref()
    rng = np.random.default_rng(1)
    kern = rng.standard_normal(k * k).astype(np.float32).astype(np.float64)
    img = rng.standard_normal((1, m * n)).astype(np.float32).astype(np.float64)
    if ref is not None:
        kind = "reference"
        t0 = time.perf_counter()
        T = ref.build(m, n, k, s, p, kern)
        build_s = time.perf_counter() - t0
        nnz = T.shape()[2]
        run = lambda: T.convolve(img, threads=cores)  # noqa: E731
    else:
        kind = "port"
        orc = oracle.Oracle()
        t0 = time.perf_counter()
        ptr, idx, val = orc.build_transform(m, n, k, s, p, kern)
        build_s = time.perf_counter() - t0
        nnz = val.size
        cores = 1
        run = lambda: orc.spmv_f64(ptr, idx, val, img[0])  # noqa: E731
    run()  # warm
    t0 = time.perf_counter()
    reps = 0
    while True:
        run()
        reps += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    single = None
    if kind == "reference" and cores > 1:  # threads=1 beside threads=nproc
        T.convolve(img, threads=1)
        s0 = time.perf_counter()
        reps1 = 0
        while time.perf_counter() - s0 < min(3.0, seconds):
            T.convolve(img, threads=1)
            reps1 += 1
        d1 = time.perf_counter() - s0
        single = {"value": nnz * reps1 / d1 / 1e9, "cores": 1, "us_per_image": d1 / reps1 * 1e6}
    return {"value": nnz * reps / dt / 1e9, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{reps} single-image convolve() calls on {m}x{n} k{k} s{s} p{p} "
                      f"({dt:.1f} s, threads={cores}); build_transform {build_s * 1e3:.0f} ms",
            "build_ms": build_s * 1e3, "us_per_image": dt / reps * 1e6, "single_thread": single}


def run_reference(args, cfg):
    """--impl reference: the reference CPU path on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    spec = cfg["spec"]
    m, n, k, s, p = spec
    cores = os.cpu_count() or 1
    ref = oracle.try_ref()
    rng = np.random.default_rng(1)
    kern = rng.standard_normal(k * k).astype(np.float32).astype(np.float64)
    imgs = rng.standard_normal((4, m * n)).astype(np.float32).astype(np.float64)
    if ref is not None:
        kind = "reference"
        T = ref.build(m, n, k, s, p, kern)
        nnz = T.shape()[2]
        step = lambda i: T.convolve(imgs[i % 4][None], threads=cores)  # noqa: E731
    else:
        kind = "port"
        orc = oracle.Oracle()
        ptr, idx, val = orc.build_transform(m, n, k, s, p, kern)
        nnz = val.size
        cores = 1
        step = lambda i: orc.spmv_f64(ptr, idx, val, imgs[i % 4])  # noqa: E731
    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i)
    dt = time.perf_counter() - t0
    value = nnz * args.steps / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"] + " -- one image per step (bounded CPU sample)",
                   "m": m, "n": n, "k": k, "s": s, "p": p, "nnz": nnz},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{args.steps} single-image convolve() steps, threads={cores}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# Our arm
# ----------------------------------------------------------------------------

def timed_build(sp, torch, kern, spec, dev, stream, reps=5, warm=3):
    """Device time of the one-time CSR build (kernel only: a GPU-side sleep
    queued first keeps the stream busy while the host enqueues the build, so
    the events bracket GPU work, not host latency) and host wall time of the call."""
    out, t = [], None
    for i in range(warm + reps):
        if t is not None:
            t.close()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        e0.record(stream)
        h0 = time.perf_counter()
        t = sp.build_transform(kern, spec, device=dev.index, stream=stream)
        h1 = time.perf_counter()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if i >= warm:
            out.append((e0.elapsed_time(e1), (h1 - h0) * 1e3))
    return t, statistics.median(x[0] for x in out), statistics.median(x[1] for x in out)


def device_steps(sp, torch, t, b, steps, warmup, dev, stream, seed):
    """Times `steps` spmm calls over a resident [b, cols] batch (CUDA events on
    the launching stream).  Inputs smaller than 2x L2 get a 512 MB scrub
    between steps, outside the events."""
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    X = torch.randn(max(b, 1), t.cols, generator=gen, device=dev, dtype=torch.float32)
    Y = torch.empty(max(b, 1), t.rows, device=dev, dtype=torch.float32)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    need_flush = 4 * b * (t.cols + t.rows) + 8 * t.nnz < 2 * l2_bytes
    scrub = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if need_flush else None
    # After the 512 MB write, a 512 MB read: L2 ends cold AND clean, so the
    # timed kernel does not pay for write-backs of the scrub's dirty lines.
    clean = torch.ones(128 << 20, dtype=torch.float32, device=dev) if need_flush else None
    sink = torch.empty((), dtype=torch.float32, device=dev) if need_flush else None

    def flush(i):
        scrub.fill_(i & 0xFF)
        torch.sum(clean, dim=0, out=sink)

    for i in range(warmup):
        if scrub is not None:
            flush(i)
        sp.spmm(t, X[:b], Y[:b], stream=stream)
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    for i in range(steps):
        if scrub is not None:
            flush(i)  # outside the events: evicts X, Y and T from L2
        ev[i][0].record(stream)
        sp.spmm(t, X[:b], Y[:b], stream=stream)
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    ms = [a.elapsed_time(c) for a, c in ev]
    l2 = ("512 MB scrub write + 512 MB clean read between steps (outside events)" if need_flush else
          f"working set larger than L2 (X+Y+T {(4 * b * (t.cols + t.rows) + 8 * t.nnz) / 1e6:.0f} MB"
          f" > 2 x {l2_bytes / 1e6:.0f} MB)")
    return X, Y, ms, l2


def secondary(sp, torch, dev, stream, steps, world=1):
    """Extras: config 4 at its per-GPU batch (8 images; at N GPUs the job is
    BASELINE's 'batch 64 over 8 B200' when N = 8: every rank times its own
    slice, max over ranks) and, at N = 1 only, config 2 (single-image SpMV,
    cold and warm L2) and config 3 in CSC layout -- kernel time, roofline
    fraction and build."""
    from paper_2411_19419_b200.shard import max_over_ranks
    out = {}
    peak, _ = peaks()
    rng = np.random.default_rng(99)
    for c in ((2, 4) if world == 1 else (4,)):
        cfg = CONFIGS[c]
        m, n, k, s, p = cfg["spec"]
        b = cfg["per_gpu_batch"]
        spec = sp.ConvSpec(m, n, k, s, p)
        kern = sp.Kernel(k, rng.standard_normal(k * k).astype(np.float32))
        t, bld_ms, _ = timed_build(sp, torch, kern, spec, dev, stream)
        X, Y, ms, l2 = device_steps(sp, torch, t, b, steps, 3, dev, stream, 7)
        alg = algorithmic_bytes(t.rows, t.cols, t.nnz, b)
        mean = max_over_ranks(sum(ms), dev) / len(ms)  # max over ranks (identity at N = 1)
        bld_ms = max_over_ranks(bld_ms, dev)
        bb = 8 * t.nnz + 4 * (t.rows + 1)
        out[f"config{c}"] = {
            "workload": cfg["name"], "batch": b, "n_gpus": world, "global_batch": b * world,
            "kernel": t.last_kernel, "ms_per_step": mean,
            "ms_min": min(ms), "value": world * b * t.nnz / (mean * 1e-3) / 1e9, "unit": UNIT,
            "gb_per_s": alg / (mean * 1e-3) / 1e9, "frac": alg / (mean * 1e-3) / 1e9 / peak,  # per GPU
            "l2": l2, "build_ms_device": bld_ms, "build_frac": bb / (bld_ms * 1e-3) / 1e9 / peak,
        }
        if c == 2:
            # warm: the paper's use (one build, repeated SpMV): 64 back-to-back
            # single-image SpMVs over 8 different images, T L2-resident,
            # chained by programmatic dependent launch
            Xw = torch.randn(8, t.cols, device=dev, dtype=torch.float32)
            Yw = torch.empty(8, t.rows, device=dev, dtype=torch.float32)
            for i in range(8):
                sp.spmm(t, Xw[i:i + 1], Yw[i:i + 1], stream=stream)
            torch.cuda.synchronize(dev)
            # one CUDA graph of the 64 launches: host enqueue cost out of the timing
            cs = torch.cuda.Stream(dev)  # graphs are captured on a side stream
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                for i in range(64):
                    sp.spmm(t, Xw[i % 8:i % 8 + 1], Yw[i % 8:i % 8 + 1], stream=cs)
            with torch.cuda.stream(cs):
                g.replay()
            torch.cuda.synchronize(dev)
            w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(cs):
                w0.record(cs)
                g.replay()
                w1.record(cs)
            torch.cuda.synchronize(dev)
            wm = w0.elapsed_time(w1) / 64
            del g
            out["config2"]["warm"] = {
                "ms_per_step": wm, "value": t.nnz / (wm * 1e-3) / 1e9, "unit": UNIT,
                "gb_per_s": alg / (wm * 1e-3) / 1e9,
                "l2": "T (13.3 MB) L2-resident: one CUDA graph of 64 back-to-back SpMVs over 8 images, "
                      "PDL-chained"}
            del Xw, Yw
        del X, Y
        t.close()
    if world > 1:
        return out
    # config 3 in CSC layout: the CSC build (CSR arrays + column-major
    # storage) and the apply through the same kernels
    cfg = CONFIGS[3]
    m, n, k, s, p = cfg["spec"]
    spec = sp.ConvSpec(m, n, k, s, p)
    kern = sp.Kernel(k, rng.standard_normal(k * k).astype(np.float32))
    cms = []
    for i in range(8):
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        e0.record(stream)
        tc = sp.build_transform(kern, spec, layout=sp.Layout.CSC, device=dev.index, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if i >= 3:
            cms.append(e0.elapsed_time(e1))
        if i < 7:
            tc.close()
    cb = 2 * 8 * tc.nnz + 4 * (tc.rows + tc.cols + 2)
    X, Y, ms, l2 = device_steps(sp, torch, tc, cfg["per_gpu_batch"], max(10, steps // 2), 3, dev, stream, 8)
    mean = statistics.mean(ms)
    alg = algorithmic_bytes(tc.rows, tc.cols, tc.nnz, cfg["per_gpu_batch"])
    out["config3_csc"] = {
        "workload": cfg["name"] + ", CSC layout", "batch": cfg["per_gpu_batch"], "kernel": tc.last_kernel,
        "build_ms_device": statistics.median(cms), "build_bytes": cb,
        "build_frac": cb / (statistics.median(cms) * 1e-3) / 1e9 / peak,
        "ms_per_step": mean, "frac": alg / (mean * 1e-3) / 1e9 / peak}
    del X, Y
    tc.close()
    return out


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2411_19419_b200 as sp
    from paper_2411_19419_b200.shard import max_over_ranks, sum_over_ranks

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # One rank per GPU.  SPCONV_B200_DIST_BACKEND=gloo (+ more ranks than GPUs,
    # ranks sharing devices) exists only to exercise the multi-rank logic on a
    # one-GPU box; the measured configuration is NCCL with one GPU per rank.
    backend = os.environ.get("SPCONV_B200_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    m, n, k, s, p = cfg["spec"]
    # Weak scaling: every rank owns a fixed slice of `b` images (the batch
    # shards with no collective); the whole job processes b * world images.
    b = args.batch or cfg["per_gpu_batch"]
    total_batch = b * world
    spec = sp.ConvSpec(m, n, k, s, p)
    rng = np.random.default_rng(1234)
    kern = sp.Kernel(k, rng.standard_normal(k * k).astype(np.float32))
    stream = torch.cuda.current_stream(dev)

    # ---- CSR build (one-time cost), device-timed: a local replica per rank ----
    t, bld_dev, bld_host = timed_build(sp, torch, kern, spec, dev, stream)
    rows, cols, nnz = t.rows, t.cols, t.nnz

    # ---- timed region: inputs resident in HBM ----
    sampler = ClockSampler(local).start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    w0 = time.perf_counter()
    X, Y, ms, l2 = device_steps(sp, torch, t, b, args.steps, args.warmup, dev, stream, 1000 + rank)
    w1 = time.perf_counter()
    if world > 1:
        dist.barrier()
    sampler.stop()
    kernel = t.last_kernel
    gather = None
    if args.gather and world > 1:
        # the optional final gather of every rank's outputs to rank 0 (NCCL
        # over NVLink), timed separately from the step: max over ranks
        from paper_2411_19419_b200.shard import gather_outputs
        dist.barrier()
        torch.cuda.synchronize(dev)
        ge0, ge1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ge0.record(stream)
        out = gather_outputs(Y[:b], total_batch)  # the result is ordered on the current stream
        ge1.record(stream)
        torch.cuda.synchronize(dev)
        g_ms = max_over_ranks(ge0.elapsed_time(ge1), dev)
        moved = 4 * (total_batch - b) * rows
        gather = {"ms": g_ms, "bytes_to_root": moved, "gb_per_s": moved / (g_ms * 1e-3) / 1e9,
                  "collective": f"torch.distributed.gather ({dist.get_backend()})"}
        del out
    launches_per_step = kernel.count("+") + 1
    elapsed_ms = sum(ms)
    max_ms = max_over_ranks(elapsed_ms, dev)
    ms_per_step = max_ms / args.steps
    value = total_batch * nnz * args.steps / (max_ms * 1e-3) / 1e9
    launch_ms = elapsed_ms / args.steps  # this rank's average step (all launches of one call)
    alg = algorithmic_bytes(rows, cols, nnz, b)
    peak, peak_src = peaks()
    achieved = alg / (launch_ms * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(args.config, b)
    clocks = sampler.summary(w0, w1)

    # ---- e2e through the C ABI with pinned host buffers ----
    e2e_steps = max(2, min(args.steps, args.e2e_steps))
    Xh = torch.empty(max(b, 1), cols, dtype=torch.float32, pin_memory=True)
    Xh.copy_(X.cpu())
    Yh = torch.empty(max(b, 1), rows, dtype=torch.float32, pin_memory=True)
    del X, Y
    sp.convolve_batch(t, Xh[:b], Yh[:b])  # warm (workspace allocation)
    if world > 1:
        dist.barrier()
    h0 = time.perf_counter()
    for _ in range(e2e_steps):
        sp.convolve_batch(t, Xh[:b], Yh[:b])
    e2e_ms = (time.perf_counter() - h0) * 1e3
    e2e_max = max_over_ranks(e2e_ms, dev)
    e2e_value = total_batch * nnz * e2e_steps / (e2e_max * 1e-3) / 1e9
    h2d = int(sum_over_ranks(4 * b * cols, dev))
    d2h = int(sum_over_ranks(4 * b * rows, dev))
    bld_bytes = 8 * nnz + 4 * (rows + 1)

    extra = None
    if not args.no_secondary:  # (collective timing at N > 1: every rank takes part)
        extra = secondary(sp, torch, dev, stream, max(10, min(args.steps, 30)), world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg["spec"], seconds=args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {
                "workload": cfg["name"], "m": m, "n": n, "k": k, "s": s, "p": p,
                "global_batch": total_batch, "per_gpu_batch": b, "rows": rows, "cols": cols,
                "nnz": nnz, "parallelism": f"batch-dp{world} (CSR replica per GPU, no collective)",
                "why_this_config": ("BASELINE metric is quoted 'at 1/2/4/8 B200': configs[2] (batch 256 of "
                                    "1024^2, sharded over 1/2/4/8); configs[1] (single 512^2 SpMV, 14.6 MB, "
                                    "L2-sized) is reported under secondary.config2 (cold and warm)")
                if args.config == 3 and not args.spec else None,
                "l2": l2,
            },
            "gb_per_s": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes": alg, "kernel": kernel,
                         "launch_ms": launch_ms, "peak_source": peak_src,
                         "traffic_source": traffic_src,
                         "note": "achieved = SURVEY 8(d) bytes of one spmm call (all its launches) / "
                                 "its CUDA-event duration"},
            "build": {"ms_device": bld_dev, "ms_host_wall": bld_host, "bytes": bld_bytes,
                      "gb_per_s": bld_bytes / (bld_dev * 1e-3) / 1e9,
                      "frac": bld_bytes / (bld_dev * 1e-3) / 1e9 / peak},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "ms_per_step": e2e_max / e2e_steps,
                    "path": "spconv_convolve_host (C ABI), pinned host buffers"},
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clocks,
            "gather": gather,
            "secondary": extra,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    t.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------------------------
# DenseNet121 layer table (paper Table 1 protocol)
# ----------------------------------------------------------------------------

PAPER_TABLE1_US = {"CSR-C (SciPy, i7-8700)": 1507.0, "CSR-T (PyTorch sparse CSR, GTX 1070)": 9187.0,
                   "CSR-G (CuPy, GTX 1070)": 11737.0, "Conv2D-G (PyTorch, GTX 1070)": 11143.0}


def reference_layer_table(trials, warmup):
    """The reference's own run_layer_bench (inc/bench.hpp:202-261) per layer on
    this host, single-threaded as the reference CLI defaults (--threads 1)."""
    import oracle
    from paper_2411_19419_b200.layers import densenet121_layers
    ref = oracle.try_ref()
    if ref is None:
        return None
    rows = []
    for i, L in enumerate(densenet121_layers()):
        rows.append(ref.run_layer_bench(L.name, L.m, L.n, L.k, L.s, L.p, trials, warmup,
                                        ref.derive_seed(42, i), 1))
    return {"layers": rows, "total_csr_us": sum(r["CSR-SpMV"][0] for r in rows),
            "total_csc_us": sum(r["CSC-SpMV"][0] for r in rows),
            "total_im2col_us": sum(r["im2col"][0] for r in rows),
            "total_csr_build_us": sum(r["CSR-SpMV"][2] for r in rows), "threads": 1,
            "kind": "reference"}


def run_densenet(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    metric = "DenseNet121 single-channel layer table: total apply time over all 123 layers (paper Table 1)"
    if args.impl == "reference":
        t0 = time.perf_counter()
        ref = reference_layer_table(args.steps, args.warmup)
        line = {"impl": "reference", "metric": metric, "unit": "us", "higher_is_better": False,
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "config": {"workload": "densenet121 layer table (123 layers)"}, "data": "synthetic",
                "dtype": "f64"}
        if ref is None:
            line["unavailable"] = "oracle/_ref not built"
        else:
            line.update(value=ref["total_csr_us"], ms_per_step=ref["total_csr_us"] / 1e3,
                        cpu_baseline={"value": ref["total_csr_us"], "unit": "us", "cores": 1,
                                      "kind": "reference",
                                      "sample": f"{args.steps} trials per layer, threads=1"},
                        e2e={"value": ref["total_csr_us"], "unit": "us", "h2d_bytes_per_step": 0,
                             "d2h_bytes_per_step": 0},
                        reference_methods={k: ref[k] for k in ("total_csr_us", "total_csc_us",
                                                               "total_im2col_us", "total_csr_build_us")},
                        wall_s=time.perf_counter() - t0)
        print(json.dumps(line), flush=True)
        return
    from paper_2411_19419_b200.layer_bench import markdown, run_table_bench
    res = run_table_bench(trials=args.steps, warmup=args.warmup)
    ref = None
    if not args.no_cpu_baseline:
        ref = reference_layer_table(min(args.steps, 100), min(args.warmup, 10))
    h2d = sum(r["m"] * r["n"] * 4 for r in res["layers"])
    d2h = sum(((r["m"] + 2 * r["p"] - r["k"]) // r["s"] + 1) * ((r["n"] + 2 * r["p"] - r["k"]) // r["s"] + 1) * 4
              for r in res["layers"])
    line = {
        "metric": metric, "value": res["total_device_us"], "unit": "us", "higher_is_better": False,
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res["total_device_us"] / 1e3, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": "densenet121 layer table (123 single-channel layers, paper Table 2)",
                   "timing": f"per layer: CUDA graph of {res['graph_reps']} SpMV launches, "
                             f"{args.steps} replays; totals = sum of per-layer means"},
        "total_device_sem_us": res["total_device_sem_us"],
        "network_graph_us": res["network_graph_us"],
        "total_build_us": res["total_build_us"],
        "e2e": {"value": res["total_host_us"], "unit": "us", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "path": "spconv_convolve_host per layer (pinned fp32 image, H2D + SpMV + D2H)"},
        "gpu_launches": len(res["layers"]),
        "paper_table1_us": PAPER_TABLE1_US,
        "cpu_baseline": None if ref is None else {
            "value": ref["total_csr_us"], "unit": "us", "cores": 1, "kind": "reference",
            "sample": "reference run_layer_bench, CSR-SpMV, threads=1",
            "csc_us": ref["total_csc_us"], "im2col_us": ref["total_im2col_us"]},
    }
    if args.report:
        with open(args.report, "w") as f:
            f.write(markdown(res, ref))
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, choices=sorted(CONFIGS), default=3)
    ap.add_argument("--batch", type=int, default=0, help="override the per-GPU batch")
    ap.add_argument("--spec", default="", help="tuning only: m,n,k,s,p replacing the config's geometry")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the config 2/4 extras")
    ap.add_argument("--gather", action="store_true",
                    help="N>1: also time the optional final gather of all outputs to rank 0")
    ap.add_argument("--workload", choices=["config", "densenet121"], default="config",
                    help="densenet121: the paper's Table 1 layer-table protocol")
    ap.add_argument("--report", default="", help="densenet121: write the per-layer markdown here")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    cfg = CONFIGS[args.config]
    if args.spec:
        spec = tuple(int(v) for v in args.spec.split(","))
        cfg = dict(cfg, spec=spec, name=f"custom spec {spec} (tuning run, not a BASELINE config)")
    if args.workload == "densenet121":
        run_densenet(args)
    elif args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
