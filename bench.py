#!/usr/bin/env python
"""Benchmark of the conv-as-SpMV hot path (BASELINE.json metric).

Workload (default, --config 3): BASELINE config 3 -- a GLOBAL batch of 256
1024x1024 fp32 images, 3x3 kernel, s=1, p=1, applied as a batched SpMM of the
CSR transform T (9,424,900 stored entries), "sharded over 1/2/4/8 B200": with
N GPUs (torchrun, one rank per GPU) rank r owns the contiguous slice
shard.batch_slice(256, r, N) (256/N images) and builds its own CSR replica;
there is no collective on the data path.  Scaling is therefore STRONG (the job
is fixed as N grows).  Config 4 (4096^2 k7 s2 p3, a global batch of 64: 8 per
GPU at N = 8) is reported beside it the same way.

Inputs are the reference's own seeded generator (inc/rng.hpp via the
library's spconv_random_normal): S = derive_seed(42, cfg), kernel =
random_normal_kernel(k, derive_seed(S, 1)), image g = random_normal_grid(m, n,
derive_seed(S, 2 + g)), rounded to fp32 -- the same data the oracle and the
reference arm see.

One step = one spconv_spmm call over this rank's slice (two launches: the
fused check-and-apply + its fixup pass at config 3), inputs resident in HBM
(config 3's 1 GB X slice is larger than the 126 MB L2, so no flush; working
sets under 2x L2 get a 512 MB scrub write + 512 MB read between steps, outside
the timed events).  Timing: barrier, synchronize, ONE CUDA-event window over
the K steps on the launching stream, synchronize; the job time is the max
over ranks of that window, cross-checked against the cross-rank wall clock
(earliest rank start after the common barrier to the last rank's end).
value = global images x nnz / job time (G nnz-MAC/s).

After timing, images {0, b/2, b-1} of every rank's slice are checked bit for
bit against the oracle's fp32 ordered-fmaf restatement (the checker, never on
the timed path): "parity" in the line.

e2e = the same metric through the C ABI (spconv_convolve_host) with pinned
HOST buffers: H2D + SpMM + D2H inside the timed region.

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
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# global_batch: the job's images, sharded over the ranks; seed = cfg index of
# SURVEY 8(d)'s derive_seed(42, cfg) (configs[0] = config 1).
CONFIGS = {
    1: dict(spec=(64, 64, 3, 1, 1), global_batch=1, seed=0, name="config1: 64x64 single image, k3 s1 p1"),
    2: dict(spec=(512, 512, 5, 2, 2), global_batch=1, seed=1,
            name="config2: 512x512 single image, k5 s2 p2 SpMV"),
    3: dict(spec=(1024, 1024, 3, 1, 1), global_batch=256, seed=2,
            name="config3: batch 256 of 1024x1024 images, k3 s1 p1, batched SpMM sharded over the GPUs"),
    4: dict(spec=(4096, 4096, 7, 2, 3), global_batch=64, seed=3,
            name="config4: batch 64 of 4096x4096 images, k7 s2 p3, build + batched SpMM sharded over the GPUs"),
}
METRIC = "SpMV-conv nnz-MAC/s (whole job) with HBM GB/s and CSR build ms"
UNIT = "G nnz-MAC/s"
BASE_SEED = 42


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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


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


def mono() -> float:
    """System-wide monotonic clock (comparable across the ranks of one node)."""
    return time.clock_gettime(time.CLOCK_MONOTONIC)


# ----------------------------------------------------------------------------
# Inputs: the reference's generator (inc/rng.hpp), via the product library
# ----------------------------------------------------------------------------

def problem_kernel(sp, cfg_idx: int, k: int) -> np.ndarray:
    """random_normal_kernel(k, derive_seed(S, 1)) rounded to fp32."""
    S = sp.derive_seed(BASE_SEED, cfg_idx)
    return sp.random_normal(sp.derive_seed(S, 1), k * k).astype(np.float32)


def problem_images(sp, cfg_idx: int, first: int, count: int, cols: int, out=None, threads: int = 16):
    """Images first .. first+count-1 of the config's global batch:
    random_normal_grid(m, n, derive_seed(S, 2 + g)) rounded to fp32, generated
    on host threads (one image per task) into `out` ([count, cols] float32)."""
    S = sp.derive_seed(BASE_SEED, cfg_idx)
    if out is None:
        out = np.empty((count, cols), np.float32)

    def one(i):
        tmp = sp.random_normal(sp.derive_seed(S, 2 + first + i), cols)
        out[i] = tmp  # fp32 rounding

    with ThreadPoolExecutor(max(1, min(threads, os.cpu_count() or 1, count))) as ex:
        list(ex.map(one, range(count)))
    return out


def pinned_images(sp, torch, cfg_idx, first, count, cols):
    Xh = torch.empty(max(count, 1), cols, dtype=torch.float32, pin_memory=True)
    problem_images(sp, cfg_idx, first, count, cols, out=Xh.numpy()[:count])
    return Xh


# ----------------------------------------------------------------------------
# Parity: the oracle's fp32 restatement is the CHECKER of what was timed
# ----------------------------------------------------------------------------

def parity_check(spec, kern, Xh, Y, which):
    """Images `which` of this rank's slice: the device output Y[i] against the
    oracle's ordered-fmaf fp32 SpMV of the oracle-built CSR (bit for bit).
    Returns (all_bitexact, worst relative deviation)."""
    from oracle import Oracle
    orc = Oracle()
    ptr, idx, val = orc.build_native(*spec, kern)
    X = np.stack([Xh[i].numpy() if hasattr(Xh[i], "numpy") else Xh[i] for i in which])
    want = orc.spmm_native(ptr, idx, val, X)
    got = np.stack([Y[i].cpu().numpy() for i in which])
    same = bool(np.array_equal(got.view(np.uint32), want.view(np.uint32)))
    dev = float(np.max(np.abs(got.astype(np.float64) - want) / np.maximum(1e-30, np.abs(want).astype(np.float64) + 1e-30)))
    return same, dev


def orc_native(spec, kern32):
    from oracle import Oracle
    return Oracle().build_native(*spec, kern32)


def spmm_oracle(ptr, idx, val, Xh, which):
    from oracle import Oracle
    X = np.stack([Xh[i].numpy() if hasattr(Xh[i], "numpy") else Xh[i] for i in which])
    return Oracle().spmm_native(ptr, idx, val, X)


def slice_probe(b: int):
    return sorted({0, b // 2, max(b - 1, 0)}) if b > 0 else []


# ----------------------------------------------------------------------------
# CPU baseline: the reference's own convolve() (oracle/_ref) on a bounded sample
# ----------------------------------------------------------------------------

def reference_inputs(ref, cfg_idx, m, n, k, count, threads):
    """The reference generator's own grids (its random_normal_grid), rounded to
    fp32 and widened back: the doubles of the fp32 values the device sees."""
    S = ref.derive_seed(BASE_SEED, cfg_idx)
    kern = ref.random_normal_kernel(k, ref.derive_seed(S, 1)).reshape(-1).astype(np.float32).astype(np.float64)
    imgs = np.empty((count, m * n), np.float64)

    def one(i):
        imgs[i] = ref.random_normal_grid(m, n, ref.derive_seed(S, 2 + i)).reshape(-1).astype(np.float32)

    with ThreadPoolExecutor(max(1, min(threads, count))) as ex:
        list(ex.map(one, range(count)))
    return kern, imgs


def cpu_baseline(cfg, seconds: float = 10.0):
    import oracle
    m, n, k, s, p = cfg["spec"]
    cores = os.cpu_count() or 1
    ref = oracle.try_ref()
    if ref is not None:
        kind = "reference"
        kern, img = reference_inputs(ref, cfg["seed"], m, n, k, 1, 1)
        t0 = time.perf_counter()
        T = ref.build(m, n, k, s, p, kern)
        build_s = time.perf_counter() - t0
        nnz = T.shape()[2]
        run = lambda: T.convolve(img, threads=cores)  # noqa: E731
    else:
        kind = "port"
        orc = oracle.Oracle()
        S = orc.derive_seed(BASE_SEED, cfg["seed"])
        kern = orc.random_normal_f32(orc.derive_seed(S, 1), k * k).astype(np.float64)
        img = orc.random_normal_f32(orc.derive_seed(S, 2), m * n).astype(np.float64)[None]
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
            "cpu": cpu_model(),
            "sample": f"{reps} single-image convolve() calls on {m}x{n} k{k} s{s} p{p} "
                      f"({dt:.1f} s, threads={cores}); build_transform {build_s * 1e3:.0f} ms",
            "build_ms": build_s * 1e3, "us_per_image": dt / reps * 1e6, "single_thread": single}


def run_reference(args, cfg):
    """--impl reference: the reference CPU path (oracle/_ref: the reference's
    own headers compiled unmodified) on this box's host cores, the same
    workload as our arm -- every step convolves the whole global batch (the
    reference has no batch API: its convolve() per image, threads = all
    cores).  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    m, n, k, s, p = cfg["spec"]
    B = args.global_batch or cfg["global_batch"]
    cores = os.cpu_count() or 1
    ref = oracle.try_ref()
    if ref is not None:
        kind = "reference"
        kern, imgs = reference_inputs(ref, cfg["seed"], m, n, k, B, cores)
        T = ref.build(m, n, k, s, p, kern)
        nnz = T.shape()[2]
        step = lambda: T.convolve(imgs, threads=cores)  # noqa: E731
    else:
        kind = "port"
        orc = oracle.Oracle()
        S = orc.derive_seed(BASE_SEED, cfg["seed"])
        kern = orc.random_normal_f32(orc.derive_seed(S, 1), k * k).astype(np.float64)
        imgs = np.stack([orc.random_normal_f32(orc.derive_seed(S, 2 + g), m * n) for g in range(B)]).astype(np.float64)
        ptr, idx, val = orc.build_transform(m, n, k, s, p, kern)
        nnz = val.size
        cores = 1
        step = lambda: [orc.spmv_f64(ptr, idx, val, x) for x in imgs]  # noqa: E731
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = B * nnz * args.steps / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "m": m, "n": n, "k": k, "s": s, "p": p, "nnz": nnz,
                   "global_batch": B, "per_step": f"convolve() over all {B} images, threads={cores}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "cpu": cpu_model(),
                         "sample": f"{args.steps} steps of {B} convolve() calls each, threads={cores}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# Our arm
# ----------------------------------------------------------------------------

def timed_build(sp, torch, kern, spec, dev, stream, reps=5, warm=3, layout=0):
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
        t = sp.build_transform(kern, spec, layout=layout, device=dev.index, stream=stream)
        h1 = time.perf_counter()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if i >= warm:
            out.append((e0.elapsed_time(e1), (h1 - h0) * 1e3))
    return t, statistics.median(x[0] for x in out), statistics.median(x[1] for x in out)


class L2Scrub:
    """512 MB write + 512 MB read between steps (outside the events): L2 ends
    cold AND clean, so a timed kernel pays neither for hits nor for write-backs."""

    def __init__(self, torch, dev):
        self.torch = torch
        self.scrub = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        self.clean = torch.ones(128 << 20, dtype=torch.float32, device=dev)
        self.sink = torch.empty((), dtype=torch.float32, device=dev)

    def __call__(self, i):
        self.scrub.fill_(i & 0xFF)
        self.torch.sum(self.clean, dim=0, out=self.sink)


def needs_flush(torch, dev, rows, cols, nnz, b):
    return 4 * b * (cols + rows) + 8 * nnz < 2 * torch.cuda.get_device_properties(dev).L2_cache_size


def l2_note(torch, dev, rows, cols, nnz, b):
    if needs_flush(torch, dev, rows, cols, nnz, b):
        return "512 MB scrub write + 512 MB clean read between steps (outside events)"
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    return (f"working set larger than L2 (X+Y+T {(4 * b * (cols + rows) + 8 * nnz) / 1e6:.0f} MB"
            f" > 2 x {l2 / 1e6:.0f} MB)")


def window_steps(torch, fn, steps, warmup, dev, stream, flush=None):
    """W untimed calls, then K timed calls.  Without a flush: ONE event window
    over the K calls (returns its total ms).  With a flush between calls:
    per-call windows (the flush stays outside), summed."""
    for i in range(warmup):
        if flush:
            flush(i)
        fn()
    torch.cuda.synchronize(dev)
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1), None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush(i)
        ev[i][0].record(stream)
        fn()
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    ms = [a.elapsed_time(c) for a, c in ev]
    return sum(ms), ms


def device_line(sp, torch, t, X, Y, b, steps, dev, stream, peak, fn=None, alg=None):
    """Kernel-side numbers of one single-GPU workload (no ranks involved)."""
    fn = fn or (lambda: sp.spmm(t, X[:b], Y[:b], stream=stream))
    flush = L2Scrub(torch, dev) if needs_flush(torch, dev, t.rows, t.cols, t.nnz, b) else None
    tot, ms = window_steps(torch, fn, steps, 3, dev, stream, flush)
    mean = tot / steps
    alg = alg if alg is not None else algorithmic_bytes(t.rows, t.cols, t.nnz, b)
    out = {"batch": b, "kernel": t.last_kernel, "ms_per_step": mean,
           "value": b * t.nnz / (mean * 1e-3) / 1e9, "unit": UNIT,
           "algorithmic_bytes": alg, "gb_per_s": alg / (mean * 1e-3) / 1e9,
           "frac": alg / (mean * 1e-3) / 1e9 / peak, "l2": l2_note(torch, dev, t.rows, t.cols, t.nnz, b)}
    if ms:
        out["ms_min"] = min(ms)
    return out


def sharded_workload(sp, torch, cfg, args, dev, stream, world, rank, steps, warmup, want_e2e):
    """One BASELINE config sharded over the ranks: build (device-timed), the K
    timed steps (max over ranks, cross-checked against the cross-rank wall
    clock), parity of the timed outputs, and (optionally) e2e through the C ABI."""
    import torch.distributed as dist

    from paper_2411_19419_b200.shard import batch_slice, max_over_ranks, sum_over_ranks
    m, n, k, s, p = cfg["spec"]
    B = args.global_batch if (args.global_batch and cfg is CONFIGS[args.config]) else cfg["global_batch"]
    first, b = batch_slice(B, rank, world)
    spec = sp.ConvSpec(m, n, k, s, p)
    kern32 = problem_kernel(sp, cfg["seed"], k)
    kern = sp.Kernel(k, kern32.astype(np.float64))
    t, bld_dev, bld_host = timed_build(sp, torch, kern, spec, dev, stream)
    rows, cols, nnz = t.rows, t.cols, t.nnz
    Xh = pinned_images(sp, torch, cfg["seed"], first, b, cols)
    X = Xh.to(dev, non_blocking=False)
    Y = torch.empty(max(b, 1), rows, device=dev, dtype=torch.float32)
    fn = (lambda: sp.spmm(t, X[:b], Y[:b], stream=stream))
    flush = L2Scrub(torch, dev) if needs_flush(torch, dev, rows, cols, nnz, b) else None

    sampler = ClockSampler(dev.index).start()
    for i in range(warmup):
        if flush:
            flush(i)
        fn()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    w0 = mono()
    p0 = time.perf_counter()
    tot, _ = window_steps(torch, fn, steps, 0, dev, stream, flush)
    w1 = mono()
    p1 = time.perf_counter()
    sampler.stop()
    ev_max = max_over_ranks(tot, dev)
    job_wall = (max_over_ranks(w1, dev) + max_over_ranks(-w0, dev)) * 1e3
    # The job time is the device time of the slowest rank; the wall clock
    # from the common barrier to the last rank's end catches ranks that did
    # not overlap (e.g. serialised on one device).  With a flush between
    # steps the wall clock also counts the flushes, so it is not comparable.
    job_ms = ev_max
    timing = "cuda-events (max over ranks)"
    if flush is None and job_wall > 1.25 * ev_max + 0.5:
        job_ms, timing = job_wall, "cross-rank wall clock (exceeds the event time: ranks did not overlap)"
    value = B * nnz * steps / (job_ms * 1e-3) / 1e9
    local_ms = tot / steps
    alg = algorithmic_bytes(rows, cols, nnz, b)
    kernel = t.last_kernel

    # ---- parity of what was timed (the oracle is the checker) ----
    which = slice_probe(b)
    same, rdev = parity_check(cfg["spec"], kern32, Xh, Y, which) if b > 0 else (True, 0.0)
    all_same = max_over_ranks(0.0 if same else 1.0, dev) == 0.0
    worst = max_over_ranks(rdev, dev)

    gather = None
    if want_e2e and getattr(args, "gather", False):
        # the optional final gather of every rank's slice on rank 0 (BASELINE
        # north_star; NCCL over NVLink), timed on its own: not part of the step
        from paper_2411_19419_b200.shard import gather_outputs
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        g0 = mono()
        full = gather_outputs(Y[:b], B)
        torch.cuda.synchronize(dev)
        g1 = mono()
        gms = (max_over_ranks(g1, dev) + max_over_ranks(-g0, dev)) * 1e3
        moved = 4 * (B - b) * rows  # bytes that reach rank 0 from the others
        gather = {"ms": gms, "bytes_to_root": moved, "gb_per_s": moved / (gms * 1e-3) / 1e9 if gms > 0 else None,
                  "backend": dist.get_backend() if world > 1 else None,
                  "ok": bool(full is None or tuple(full.shape) == (B, rows))}
        del full
    e2e = None
    if want_e2e:
        Yh = torch.empty(max(b, 1), rows, dtype=torch.float32, pin_memory=True)
        sp.convolve_batch(t, Xh[:b], Yh[:b])  # warm (workspace allocation)
        e2e_steps = max(2, min(steps, args.e2e_steps))
        if world > 1:
            dist.barrier()
        h0 = mono()
        for _ in range(e2e_steps):
            sp.convolve_batch(t, Xh[:b], Yh[:b])
        h1 = mono()
        e2e_ms = (max_over_ranks(h1, dev) + max_over_ranks(-h0, dev)) * 1e3
        e2e = {"value": B * nnz * e2e_steps / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(sum_over_ranks(4 * b * cols, dev)),
               "d2h_bytes_per_step": int(sum_over_ranks(4 * b * rows, dev)),
               "steps": e2e_steps, "ms_per_step": e2e_ms / e2e_steps,
               "path": "spconv_convolve_host (C ABI), pinned host buffers, cross-rank wall clock"}
        e2e_ok = np.array_equal(Yh[which].numpy().view(np.uint32), Y[which].cpu().numpy().view(np.uint32))
        e2e["parity"] = "bitexact (== the device-timed outputs)" if max_over_ranks(0.0 if e2e_ok else 1.0, dev) == 0.0 else "MISMATCH"
        del Yh
    res = {
        "t": t, "B": B, "b": b, "rows": rows, "cols": cols, "nnz": nnz, "kernel": kernel,
        "value": value, "job_ms": job_ms, "ev_max_ms": ev_max, "job_wall_ms": job_wall, "timing": timing,
        "local_ms": local_ms, "alg": alg, "bld_dev": max_over_ranks(bld_dev, dev), "bld_host": bld_host,
        "parity": "bitexact" if all_same else "MISMATCH", "parity_images": which, "gather": gather,
        "parity_max_rel_dev": worst, "e2e": e2e, "clocks": sampler.summary(p0, p1),
        "l2": l2_note(torch, dev, rows, cols, nnz, b),
    }
    del X, Y, Xh
    return res


def secondary_single(sp, torch, dev, stream, steps, peak):
    """N = 1 only: the per-rank workloads of the N = 2/4/8 runs on one GPU
    (strong-scaling proxies), config 2's single-image SpMV (cold and warm L2),
    and config 4's per-rank slice at N = 8."""
    out = {}
    # ---- config 3 per-rank slices at N = 2 / 4 / 8 ----
    cfg = CONFIGS[3]
    m, n, k, s, p = cfg["spec"]
    kern32 = problem_kernel(sp, cfg["seed"], k)
    t = sp.build_transform(sp.Kernel(k, kern32.astype(np.float64)), sp.ConvSpec(m, n, k, s, p),
                           device=dev.index, stream=stream)
    Xh = pinned_images(sp, torch, cfg["seed"], 0, 256, t.cols)
    X = Xh.to(dev)
    Y = torch.empty(256, t.rows, device=dev)
    prox = {}
    for g, b in ((2, 128), (4, 64), (8, 32)):
        line = device_line(sp, torch, t, X, Y, b, steps, dev, stream, peak)
        line["as_rank_of"] = f"N={g}: batch_slice(256, r, {g}) = {b} images"
        prox[f"n{g}"] = line
    out["config3_per_rank_proxy"] = prox
    t.close()
    # ---- config 3 as a CSC transform (the reference's second layout): the
    # handle holds the CSC storage only and every call streams it (CSC band
    # check); algorithmic bytes 8 nnz + 4 (cols + 1) + 4 b (cols + rows)
    tc = sp.build_transform(sp.Kernel(k, kern32.astype(np.float64)), sp.ConvSpec(m, n, k, s, p), layout=1,
                            device=dev.index, stream=stream)
    alg = 8 * tc.nnz + 4 * (tc.cols + 1) + 4 * 256 * (tc.cols + tc.rows)
    line = device_line(sp, torch, tc, X, Y, 256, steps, dev, stream, peak, alg=alg)
    same, _ = parity_check(cfg["spec"], kern32, Xh, Y, slice_probe(256))
    line.update(parity="bitexact" if same else "MISMATCH", storage_bytes=tc.storage_bytes,
                storage_bytes_csr_handle=8 * tc.nnz + 4 * (tc.rows + 1),
                layout="csc (col_ptr / row_idx / vals only)")
    out["config3_csc"] = line
    tc.close()
    del X, Y
    # ---- config 3 in the reference's own arithmetic (fp64 images, per-entry
    # double multiply then add: spconv_spmm_f64, bit-identical to the
    # reference's convolve()); bytes 8 nnz + 4 (rows + 1) + 8 b (cols + rows)
    # (the check streams col_idx + fp32 vals; the exact taps are applied)
    t64 = sp.build_transform(sp.Kernel(k, kern32.astype(np.float64)), sp.ConvSpec(m, n, k, s, p),
                             device=dev.index, stream=stream)
    X64 = Xh.to(dev).double()
    Y64 = torch.empty(256, t64.rows, device=dev, dtype=torch.float64)
    alg = 8 * t64.nnz + 4 * (t64.rows + 1) + 8 * 256 * (t64.cols + t64.rows)
    line = device_line(sp, torch, t64, X64, Y64, 256, steps, dev, stream, peak, alg=alg,
                       fn=lambda: sp.spmm_f64(t64, X64, Y64, stream=stream))
    line["kernel"] = t64.last_kernel
    from oracle import Oracle
    orc = Oracle()
    ptr, idx, val = orc.build_transform(m, n, k, s, p, kern32.astype(np.float64))
    same = all(np.array_equal(Y64[i].cpu().numpy().view(np.uint64),
                              orc.spmv_f64(ptr, idx, val, X64[i].cpu().numpy()).view(np.uint64))
               for i in slice_probe(256))
    # e2e: the drop-in call shape (fp64 host buffers through spconv_convolve_host_f64)
    Xh64 = Xh.double().pin_memory()
    Yh64 = torch.empty(256, t64.rows, dtype=torch.float64).pin_memory()
    sp.convolve_batch_f64(t64, Xh64, Yh64)
    h0 = time.perf_counter()
    sp.convolve_batch_f64(t64, Xh64, Yh64)
    e2e_ms = (time.perf_counter() - h0) * 1e3
    line.update(parity="bitexact (vs the fp64 restatement of spmv_csr_rows)" if same else "MISMATCH",
                dtype="f64", e2e={"value": 256 * t64.nnz / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "ms": e2e_ms,
                                  "h2d_bytes_per_step": 8 * 256 * t64.cols, "d2h_bytes_per_step": 8 * 256 * t64.rows,
                                  "path": "spconv_convolve_host_f64 (C ABI), pinned fp64 host buffers"})
    out["config3_f64"] = line
    t64.close()
    del X64, Y64, Xh64, Yh64, Xh
    # ---- config 4: the per-rank slice at N = 8 (8 images) ----
    cfg = CONFIGS[4]
    m, n, k, s, p = cfg["spec"]
    kern32 = problem_kernel(sp, cfg["seed"], k)
    t = sp.build_transform(sp.Kernel(k, kern32.astype(np.float64)), sp.ConvSpec(m, n, k, s, p),
                           device=dev.index, stream=stream)
    Xh = pinned_images(sp, torch, cfg["seed"], 0, 8, t.cols)
    X = Xh.to(dev)
    Y = torch.empty(8, t.rows, device=dev)
    line = device_line(sp, torch, t, X, Y, 8, steps, dev, stream, peak)
    line["as_rank_of"] = "N=8: batch_slice(64, r, 8) = 8 images"
    out["config4_per_rank_proxy_n8"] = line
    del X, Y, Xh
    t.close()
    # ---- off the BASELINE shapes: config 5's widest geometry (257 x 193, k11
    # s1 p10: odd width -> cp.async element staging; 121 FMAs an output)
    # and config 3's matrix uploaded as a generic CSR (no conv geometry: the
    # row-block kernel) -- 256 images each
    for name, spec, generic in (("config5_k11", (257, 193, 11, 1, 10), False),
                                ("config3_generic_csr", (1024, 1024, 3, 1, 1), True)):
        mm, nn, kk, ss, pp = spec
        kv = problem_kernel(sp, 4 if not generic else 2, kk)
        tt = sp.build_transform(sp.Kernel(kk, kv.astype(np.float64)), sp.ConvSpec(*spec), device=dev.index,
                                stream=stream)
        if generic:
            ptr, idx, val = tt.export()
            tt.close()
            tt = sp.Transform.from_host(1024 * 1024, 1024 * 1024, ptr, idx, val, device=dev.index)
        Xh = pinned_images(sp, torch, 4 if not generic else 2, 0, 256, tt.cols)
        X = Xh.to(dev)
        Y = torch.empty(256, tt.rows, device=dev)
        line = device_line(sp, torch, tt, X, Y, 256, steps, dev, stream, peak)
        line["workload"] = f"{spec}, 256 images" + (" (uploaded as a generic CSR)" if generic else "")
        line["gflop_per_s"] = 2 * 256 * tt.nnz / (line["ms_per_step"] * 1e-3) / 1e9
        if not generic:
            ptr, idx, val = orc_native(spec, kv)
            want = spmm_oracle(ptr, idx, val, Xh, slice_probe(256))
            got = np.stack([Y[i].cpu().numpy() for i in slice_probe(256)])
            line["parity"] = "bitexact" if np.array_equal(got.view(np.uint32), want.view(np.uint32)) else "MISMATCH"
        out[name] = line
        del X, Y, Xh
        tt.close()
    # ---- config 2: one 512^2 image (cold L2) + the warm-L2 repeated SpMV ----
    cfg = CONFIGS[2]
    m, n, k, s, p = cfg["spec"]
    kern32 = problem_kernel(sp, cfg["seed"], k)
    spec = sp.ConvSpec(m, n, k, s, p)
    kern = sp.Kernel(k, kern32.astype(np.float64))
    t, bld_ms, _ = timed_build(sp, torch, kern, spec, dev, stream)
    Xh = pinned_images(sp, torch, cfg["seed"], 0, 8, t.cols)
    Xw = Xh.to(dev)
    Yw = torch.empty(8, t.rows, device=dev)
    line = device_line(sp, torch, t, Xw, Yw, 1, max(steps, 30), dev, stream, peak)
    bb = 8 * t.nnz + 4 * (t.rows + 1)
    line.update(workload=cfg["name"], build_ms_device=bld_ms, build_frac=bb / (bld_ms * 1e-3) / 1e9 / peak)
    same, _ = parity_check(cfg["spec"], kern32, Xh, Yw, [0])
    line["parity"] = "bitexact" if same else "MISMATCH"
    # warm: the paper's use (one build, repeated SpMV): one CUDA graph of 64
    # back-to-back single-image SpMVs over 8 images, T L2-resident, PDL-chained
    cs = torch.cuda.Stream(dev)
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
    alg = algorithmic_bytes(t.rows, t.cols, t.nnz, 1)
    line["warm"] = {"ms_per_step": wm, "value": t.nnz / (wm * 1e-3) / 1e9, "unit": UNIT,
                    "gb_per_s": alg / (wm * 1e-3) / 1e9,
                    "l2": "T (13.3 MB) L2-resident: one CUDA graph of 64 back-to-back SpMVs over 8 images, PDL-chained"}
    out["config2"] = line
    del Xw, Yw, Xh
    t.close()
    return out


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2411_19419_b200 as sp

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
    stream = torch.cuda.current_stream(dev)
    peak, peak_src = peaks()
    m, n, k, s, p = cfg["spec"]

    main = sharded_workload(sp, torch, cfg, args, dev, stream, world, rank, args.steps, args.warmup, True)
    t = main["t"]
    b, B = main["b"], main["B"]
    achieved = main["alg"] / (main["local_ms"] * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(args.config, b)
    bld_bytes = 8 * main["nnz"] + 4 * (main["rows"] + 1)
    launches_per_step = main["kernel"].count("+") + 1

    extra = {}
    if not args.no_secondary:
        if args.config != 4:  # BASELINE config 4 sharded the same way (every rank takes part)
            c4 = sharded_workload(sp, torch, CONFIGS[4], args, dev, stream, world, rank,
                                  max(10, min(args.steps, 30)), 3, False)
            c4b = 8 * c4["nnz"] + 4 * (c4["rows"] + 1)
            extra["config4"] = {
                "workload": CONFIGS[4]["name"], "global_batch": c4["B"], "per_gpu_batch": c4["b"],
                "n_gpus": world, "kernel": c4["kernel"], "ms_per_step": c4["job_ms"] / max(10, min(args.steps, 30)),
                "value": c4["value"], "unit": UNIT, "timing": c4["timing"], "job_wall_ms": c4["job_wall_ms"],
                "gb_per_s_per_gpu": c4["alg"] / (c4["local_ms"] * 1e-3) / 1e9,
                "frac": c4["alg"] / (c4["local_ms"] * 1e-3) / 1e9 / peak,
                "algorithmic_bytes_per_gpu": c4["alg"], "l2": c4["l2"],
                "build_ms_device": c4["bld_dev"], "build_frac": c4b / (c4["bld_dev"] * 1e-3) / 1e9 / peak,
                "parity": c4["parity"], "parity_images": c4["parity_images"]}
            c4["t"].close()
        if world == 1:
            extra.update(secondary_single(sp, torch, dev, stream, max(10, min(args.steps, 30)), peak))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, seconds=args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["job_ms"] / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (the reference's seeded generator, inc/rng.hpp)",
            "config": {
                "workload": cfg["name"], "m": m, "n": n, "k": k, "s": s, "p": p,
                "global_batch": B, "per_gpu_batch": b, "rows": main["rows"], "cols": main["cols"],
                "nnz": main["nnz"],
                "parallelism": f"batch-dp{world}: shard.batch_slice({B}, rank, {world}), CSR replica per GPU, "
                               "no collective",
                "why_this_config": ("BASELINE metric is quoted 'at 1/2/4/8 B200': configs[2] (batch 256 of "
                                    "1024^2, sharded over 1/2/4/8); configs[1] (single 512^2 SpMV, 14.6 MB, "
                                    "L2-sized) is reported under secondary.config2 (cold and warm)")
                if args.config == 3 else None,
                "l2": main["l2"],
            },
            "timing": {"method": main["timing"], "event_max_ms": main["ev_max_ms"],
                       "job_wall_ms": main["job_wall_ms"],
                       "wall_over_event": main["job_wall_ms"] / main["ev_max_ms"] if main["ev_max_ms"] else None},
            "parity": main["parity"],
            "parity_detail": {"images_per_rank": main["parity_images"], "max_rel_dev": main["parity_max_rel_dev"],
                              "against": "oracle/spconv_oracle.c fp32 ordered-fmaf SpMV of the oracle-built CSR"},
            "gb_per_s": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes": main["alg"], "kernel": main["kernel"],
                         "launch_ms": main["local_ms"], "peak_source": peak_src,
                         "traffic_source": traffic_src,
                         "note": "achieved = SURVEY 8(d) bytes of one spmm call over rank 0's slice (all its "
                                 "launches) / its CUDA-event duration"},
            "build": {"ms_device": main["bld_dev"], "ms_host_wall": main["bld_host"], "bytes": bld_bytes,
                      "gb_per_s": bld_bytes / (main["bld_dev"] * 1e-3) / 1e9,
                      "frac": bld_bytes / (main["bld_dev"] * 1e-3) / 1e9 / peak},
            "e2e": main["e2e"],
            "gather": main["gather"],
            "gpu_launches": args.steps * launches_per_step,
            "clocks": main["clocks"],
            "secondary": extra or None,
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
                                      "kind": "reference", "cpu": cpu_model(),
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
        "ms_per_step": res["total_device_us"] / 1e3, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": "densenet121 layer table (123 single-channel layers, paper Table 2)",
                   "timing": f"per layer: CUDA graph of {res['graph_reps']} SpMV launches, "
                             f"{args.steps} replays; totals = sum of per-layer means"},
        "total_device_sem_us": res["total_device_sem_us"],
        "total_csc_device_us": res["total_csc_device_us"],
        "network_graph_us": res["network_graph_us"],
        "network_group_us": res["network_group_us"],
        "total_build_us": res["total_build_us"],
        "e2e": {"value": res["e2e_group_us"], "unit": "us", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "path": "spconv_convolve_host_group (C ABI): the 123 pageable host images in, 123 outputs "
                        "out, one call (host pack, one H2D, one grouped SpMV launch, one D2H, unpack)",
                "python_api_us": res["e2e_group_python_us"]},
        "e2e_f64": {"value": res["e2e_group_f64_us"], "unit": "us", "h2d_bytes_per_step": 2 * h2d,
                    "d2h_bytes_per_step": 2 * d2h,
                    "path": "spconv_convolve_host_group_f64 (C ABI): the reference's fp64 arithmetic, every "
                            "layer's output bit-identical to its per-layer fp64 SpMV (= the reference's convolve)"},
        "e2e_per_layer": {"value": res["total_host_us"], "unit": "us", "h2d_bytes_per_step": h2d,
                          "d2h_bytes_per_step": d2h,
                          "path": "spconv_convolve_host per layer (pinned fp32 image, H2D + SpMV + D2H), "
                                  "summed over the 123 layers"},
        "gpu_launches": len(res["layers"]),
        "paper_table1_us": PAPER_TABLE1_US,
        "cpu_baseline": None if ref is None else {
            "value": ref["total_csr_us"], "unit": "us", "cores": 1, "kind": "reference", "cpu": cpu_model(),
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
    ap.add_argument("--global-batch", type=int, default=0, help="override the config's global batch")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the extra workloads")
    ap.add_argument("--gather", action="store_true", help="also time the optional final gather on rank 0")
    ap.add_argument("--workload", choices=["config", "densenet121"], default="config",
                    help="densenet121: the paper's Table 1 layer-table protocol")
    ap.add_argument("--report", default="", help="densenet121: write the per-layer markdown here")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    cfg = CONFIGS[args.config]
    if args.workload == "densenet121":
        run_densenet(args)
    elif args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
