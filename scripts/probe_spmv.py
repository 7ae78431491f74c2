"""Latency SpMV A/B (batch 1): windowed kernel (stage=window) vs the
bulk-staged kernel (stage=bulk), cold (512 MB scrub write + read between
calls, outside the events) and warm (CUDA graph of 64 PDL-chained calls)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402

dev = torch.device("cuda", 0)
scrub = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
clean = torch.ones(128 << 20, dtype=torch.float32, device=dev)
sink = torch.empty((), dtype=torch.float32, device=dev)
out = {}
for spec in ((512, 512, 5, 2, 2), (56, 56, 3, 1, 1), (224, 224, 7, 2, 3), (28, 28, 1, 1, 0), (112, 112, 3, 2, 1)):
    m, n, k, s, p = spec
    kern = np.random.default_rng(0).standard_normal(k * k).astype(np.float32)
    t = sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec))
    X = torch.randn(8, t.cols, device=dev)
    Y = torch.empty(8, t.rows, device=dev)
    for stage in ("window", "bulk"):
        with sp.options(stage=stage):
            st = torch.cuda.current_stream(dev)
            for _ in range(3):
                sp.spmm(t, X[:1], Y[:1])
            cold = []
            for i in range(30):
                scrub.fill_(i & 0xFF)
                torch.sum(clean, dim=0, out=sink)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sp.spmm(t, X[i % 8:i % 8 + 1], Y[i % 8:i % 8 + 1])
                e1.record()
                torch.cuda.synchronize()
                cold.append(e0.elapsed_time(e1) * 1e3)
            cs = torch.cuda.Stream(dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                for i in range(64):
                    sp.spmm(t, X[i % 8:i % 8 + 1], Y[i % 8:i % 8 + 1], stream=cs)
            with torch.cuda.stream(cs):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(cs):
                e0.record(cs)
                g.replay()
                e1.record(cs)
            torch.cuda.synchronize()
            warm = e0.elapsed_time(e1) * 1e3 / 64
            del g
            key = f"{spec} {stage}"
            out[key] = {"kernel": t.last_kernel, "cold_us_median": float(np.median(cold)), "warm_us": warm}
            print(key, out[key], flush=True)
    t.close()
json.dump(out, open("gpurun_out/probes/probe_spmv.json" if __import__("os").path.isdir("gpurun_out/probes") else "gpurun_out/probe_spmv.json", "w"), indent=1)
