"""A/B of the band forms at BASELINE config 3 / 4 per-GPU batches: fused
check-and-apply vs separate check kernel + apply (option fused=1 / 0), CSR and
CSC storage.  CUDA-event mean over `reps` back-to-back calls."""
import json
import sys

import numpy as np
import torch

import os  # noqa: E402

sys.path.insert(0, os.environ.get("AB_PKG", "."))  # (AB_PKG: another build of the package, for A/B runs)
import paper_2411_19419_b200 as sp  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
only = sys.argv[2] if len(sys.argv) > 2 else ""
out = {}
for spec, batches in (((1024, 1024, 3, 1, 1), (256, 128, 64, 32, 16)), ((4096, 4096, 7, 2, 3), (64, 8))):
    m, n, k, s, p = spec
    kern = np.random.default_rng(0).standard_normal(k * k).astype(np.float32)
    for layout in (0, 1):
        if only and only != ("csc" if layout else "csr"):
            continue
        t = sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec), layout=layout)
        bmax = max(batches)
        X = torch.randn(bmax, t.cols, device="cuda")
        Y = torch.empty(bmax, t.rows, device="cuda")
        for b in batches:
            row = {}
            for form in ("auto", "0", "1"):
                with sp.options(fused=form):
                    for _ in range(3):
                        sp.spmm(t, X[:b], Y[:b])
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(reps):
                        sp.spmm(t, X[:b], Y[:b])
                    e1.record()
                    torch.cuda.synchronize()
                row[form] = (round(e0.elapsed_time(e1) / reps * 1e3, 1), t.last_kernel)
            key = f"{spec} {'csc' if layout else 'csr'} b={b}"
            out[key] = row
            print(key, row, flush=True)
        del X, Y
        t.close()
json.dump(out, open(os.environ.get("AB_OUT", "gpurun_out/ab_fused.json"), "w"), indent=1)
