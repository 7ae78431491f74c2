"""SpMM speed off the band instantiations (and off TMA-describable rows): the
config-5 geometries on 257 x 193 at batch 256, other (k, s) at 1024^2, and
config 3's matrix uploaded as a generic CSR.  CUDA-event mean of `reps`
back-to-back calls; algorithmic bytes 8 nnz + 4 (rows + 1) + 4 b (cols + rows)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6466.0
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
which = sys.argv[2] if len(sys.argv) > 2 else "all"
out = {}


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cases = [((257, 193, 11, 1, 10), 256), ((257, 193, 5, 3, 4), 256), ((257, 193, 3, 2, 1), 256),
         ((257, 193, 1, 1, 0), 256), ((256, 192, 11, 1, 10), 256), ((1024, 1024, 7, 1, 3), 64),
         ((1024, 1024, 1, 1, 0), 256), ((1024, 1024, 3, 3, 1), 256), ((1024, 1024, 5, 3, 2), 256),
         ((1024, 1024, 11, 1, 5), 32)]
for spec, b in cases:
    if which != "all" and which not in str(spec):
        continue
    m, n, k, s, p = spec
    kern = np.random.default_rng(0).standard_normal(k * k).astype(np.float32)
    t = sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec))
    X = torch.randn(b, t.cols, device="cuda")
    Y = torch.empty(b, t.rows, device="cuda")
    ms = timeit(lambda: sp.spmm(t, X, Y))
    alg = 8 * t.nnz + 4 * (t.rows + 1) + 4 * b * (t.cols + t.rows)
    out[f"{spec} b={b}"] = {"ms": ms, "frac": alg / (ms * 1e-3) / 1e9 / peak, "kernel": t.last_kernel}
    print(f"{spec} b={b}", out[f"{spec} b={b}"], flush=True)
    del X, Y
    t.close()
# config 3's matrix as a generic CSR (no conv geometry): the row-block kernel
spec = (1024, 1024, 3, 1, 1)
kern = np.random.default_rng(0).standard_normal(9).astype(np.float32)
t = sp.build_transform(sp.Kernel(3, kern), sp.ConvSpec(*spec))
ptr, idx, val = t.export()
g = sp.Transform.from_host(t.rows, t.cols, ptr, idx, val)
for b in (256, 32):
    X = torch.randn(b, g.cols, device="cuda")
    Y = torch.empty(b, g.rows, device="cuda")
    ms = timeit(lambda: sp.spmm(g, X, Y))
    alg = 8 * g.nnz + 4 * (g.rows + 1) + 4 * b * (g.cols + g.rows)
    out[f"generic config3 b={b}"] = {"ms": ms, "frac": alg / (ms * 1e-3) / 1e9 / peak, "kernel": g.last_kernel}
    print(f"generic config3 b={b}", out[f"generic config3 b={b}"], flush=True)
json.dump(out, open("gpurun_out/probe_geoms.json", "w"), indent=1)
