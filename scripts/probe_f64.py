"""Times spconv_spmm_f64 (the reference-arithmetic apply) at BASELINE config 3
shapes: fp32-representable taps (vals widened) and exact double taps (vals64)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6466.0
dev = torch.device("cuda", 0)
out = {}
for spec, batches in (((1024, 1024, 3, 1, 1), (32, 256)), ((4096, 4096, 7, 2, 3), (8,)), ((512, 512, 5, 2, 2), (1,))):
    m, n, k, s, p = spec
    rng = np.random.default_rng(1)
    for exact in (False, True):
        kern = rng.standard_normal(k * k)
        if not exact:
            kern = kern.astype(np.float32).astype(np.float64)
        for layout in (0, 1):
            t = sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec), layout=layout)
            for b in batches:
                X = torch.randn(b, t.cols, dtype=torch.float64, device=dev)
                Y = torch.empty(b, t.rows, dtype=torch.float64, device=dev)
                for _ in range(3):
                    sp.spmm_f64(t, X, Y)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 10
                e0.record()
                for _ in range(reps):
                    sp.spmm_f64(t, X, Y)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                vb = 12 if exact else 8
                alg = vb * t.nnz + 4 * ((t.cols if layout else t.rows) + 1) + 8 * b * (t.cols + t.rows)
                key = f"{spec} b={b} exact={exact} layout={'csc' if layout else 'csr'}"
                out[key] = {"ms": ms, "frac": alg / (ms * 1e-3) / 1e9 / peak, "kernel": t.last_kernel}
                print(key, out[key], flush=True)
                del X, Y
            t.close()
json.dump(out, open("gpurun_out/probe_f64.json", "w"), indent=1)
