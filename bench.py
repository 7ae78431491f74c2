#!/usr/bin/env python
"""Benchmark of the conv-as-SpMV hot path (BASELINE.json metric).

Workload (default, --config 3): BASELINE config 3 -- a global batch of 256
1024x1024 fp32 images, 3x3 kernel, s=1, p=1, applied as a batched SpMM of the
CSR transform T (9,424,900 stored entries).  With N GPUs (torchrun, one rank
per GPU) every rank builds its own CSR replica on its device and owns a
contiguous slice of the batch; there is no collective on the data path.

One step = one SpMM launch over this rank's batch slice, inputs resident in
HBM (each X slice is larger than the 126 MB L2, so no flush is needed; for
--config 2, whose working set fits in L2, a 512 MB scrub runs between steps
outside the timed events).  value = whole-job nnz-MACs per second (total
images x nnz / max-over-ranks device time).  e2e = the same metric through the
C ABI with pinned HOST buffers (H2D + SpMM + D2H pipelined in the library).

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

CONFIGS = {
    1: dict(spec=(64, 64, 3, 1, 1), batch=1, name="config1: 64x64 single image, k3 s1 p1"),
    2: dict(spec=(512, 512, 5, 2, 2), batch=1, name="config2: 512x512 single image, k5 s2 p2 SpMV"),
    3: dict(spec=(1024, 1024, 3, 1, 1), batch=256,
            name="config3: batch 256 of 1024x1024 images, k3 s1 p1, batched SpMM"),
    4: dict(spec=(4096, 4096, 7, 2, 3), batch=64,
            name="config4: batch 64 of 4096x4096 images, k7 s2 p3, build + batched SpMM"),
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


def ncu_traffic(cfg: int):
    """dram bytes per launch of the SpMM kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            j = json.load(f)
        e = j.get(f"config{cfg}")
        return (float(e["dram_bytes_per_launch"]), e.get("source")) if e else (None, None)
    except Exception:
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
    return {"value": nnz * reps / dt / 1e9, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{reps} single-image convolve() calls on {m}x{n} k{k} s{s} p{p} "
                      f"({dt:.1f} s, threads={cores}); build_transform {build_s * 1e3:.0f} ms",
            "build_ms": build_s * 1e3, "us_per_image": dt / reps * 1e6}


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
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
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

def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2411_19419_b200 as sp
    from paper_2411_19419_b200.shard import batch_slice, max_over_ranks, sum_over_ranks

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    m, n, k, s, p = cfg["spec"]
    total_batch = args.batch or cfg["batch"]
    b0, b = batch_slice(total_batch, rank, world)
    spec = sp.ConvSpec(m, n, k, s, p)
    rng = np.random.default_rng(1234)
    kern = sp.Kernel(k, rng.standard_normal(k * k).astype(np.float32))
    stream = torch.cuda.current_stream(dev)

    # ---- CSR build (one-time cost), device-timed ----
    build_ms = []
    t = None
    for i in range(3 + 5):
        if t is not None:
            t.close()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record(stream)
        t = sp.build_transform(kern, spec, device=local, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if i >= 3:
            build_ms.append((e0.elapsed_time(e1), (time.perf_counter() - h0) * 1e3))
    rows, cols, nnz = t.rows, t.cols, t.nnz

    # ---- inputs resident in HBM ----
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    X = torch.randn(max(b, 1), cols, generator=gen, device=dev, dtype=torch.float32)
    Y = torch.empty(max(b, 1), rows, device=dev, dtype=torch.float32)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    need_flush = 4 * b * cols < 2 * l2_bytes
    scrub = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if need_flush else None

    def step():
        sp.spmm(t, X[:b], Y[:b], stream=stream)

    for _ in range(args.warmup):
        if scrub is not None:
            scrub.fill_(1)
        step()
    sampler = ClockSampler(local).start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    w0 = time.perf_counter()
    for i in range(args.steps):
        if scrub is not None:
            scrub.fill_(i & 0xFF)  # outside the events: evicts X, Y and T from L2
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    w1 = time.perf_counter()
    if world > 1:
        dist.barrier()
    sampler.stop()
    elapsed_ms = sum(a.elapsed_time(c) for a, c in ev)
    max_ms = max_over_ranks(elapsed_ms, dev)
    ms_per_step = max_ms / args.steps
    macs = total_batch * nnz * args.steps
    value = macs / (max_ms * 1e-3) / 1e9
    launch_ms = elapsed_ms / args.steps  # this rank's average launch duration
    alg = algorithmic_bytes(rows, cols, nnz, b)
    peak, peak_src = peaks()
    achieved = alg / (launch_ms * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(args.config)
    clocks = sampler.summary(w0, w1)

    # ---- e2e through the C ABI with pinned host buffers ----
    e2e_steps = max(2, min(args.steps, args.e2e_steps))
    Xh = torch.empty(max(b, 1), cols, dtype=torch.float32, pin_memory=True)
    Xh.copy_(X.cpu())
    Yh = torch.empty(max(b, 1), rows, dtype=torch.float32, pin_memory=True)
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

    bld_dev = statistics.median(x[0] for x in build_ms)
    bld_host = statistics.median(x[1] for x in build_ms)
    bld_bytes = 8 * nnz + 4 * (rows + 1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg["spec"], seconds=args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {
                "workload": cfg["name"], "m": m, "n": n, "k": k, "s": s, "p": p,
                "global_batch": total_batch, "per_gpu_batch": b, "rows": rows, "cols": cols,
                "nnz": nnz, "parallelism": f"batch-dp{world} (CSR replica per GPU, no collective)",
                "l2": ("512 MB scrub between steps (outside events)" if need_flush else
                       f"inputs larger than L2 (X slice {4 * b * cols / 1e6:.0f} MB > "
                       f"{l2_bytes / 1e6:.0f} MB)"),
            },
            "gb_per_s": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes": alg, "kernel": "conv_spmm_tiled",
                         "launch_ms": launch_ms, "peak_source": peak_src,
                         "traffic_source": traffic_src},
            "build": {"ms_device": bld_dev, "ms_host_wall": bld_host, "bytes": bld_bytes,
                      "gb_per_s": bld_bytes / (bld_dev * 1e-3) / 1e9,
                      "frac": bld_bytes / (bld_dev * 1e-3) / 1e9 / peak},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "ms_per_step": e2e_max / e2e_steps,
                    "path": "spconv_convolve_host (C ABI), pinned host buffers"},
            "gpu_launches": args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    t.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, choices=sorted(CONFIGS), default=3)
    ap.add_argument("--batch", type=int, default=0, help="override the global batch")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
