#!/usr/bin/env python
"""A/B of the build kernels: device time of the CSR and CSC builds (median of
N, CUDA events behind a GPU sleep so host enqueue latency is excluded) per
SPCONV_B200_BUILD setting.   python scripts/build_ab.py [N]"""
import os
import statistics
import subprocess
import sys

CODE = r'''
import statistics, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp
N = int(sys.argv[1])
st = torch.cuda.Stream()
for name, spec in (("c3", (1024, 1024, 3, 1, 1)), ("c2", (512, 512, 5, 2, 2)), ("c4", (4096, 4096, 7, 2, 3))):
    k = spec[2]
    kern = sp.Kernel(k, np.random.default_rng(0).standard_normal(k * k).astype(np.float32))
    for layout in (0, 1):
        ts = []
        for i in range(N + 3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                torch.cuda._sleep(2_000_000)
                e0.record(st)
                t = sp.build_transform(kern, sp.ConvSpec(*spec), layout=layout, stream=st)
                e1.record(st)
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
            t.close()
        print(f"{name} {'csc' if layout else 'csr'} {statistics.median(ts):8.1f} us  (min {min(ts):.1f})")
'''

n = sys.argv[1] if len(sys.argv) > 1 else "20"
for v in ("block", "persist"):
    env = dict(os.environ, SPCONV_B200_BUILD=v)
    r = subprocess.run([sys.executable, "-c", CODE, n], env=env, capture_output=True, text=True)
    for ln in r.stdout.splitlines():
        print(f"{v:8s} {ln}")
    if r.returncode:
        print(r.stderr[-2000:])
