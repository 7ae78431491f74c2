"""Anatomy of the grouped host call over the DenseNet121 table: the Python
wrapper (convolve_group) against the bare C-ABI call with prebuilt pointer
arrays, and the device time of the grouped launch."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402
from paper_2411_19419_b200.layers import densenet121_layers  # noqa: E402


def per_call(fn, n=300):
    for _ in range(30):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


ts, imgs = [], []
for li, L in enumerate(densenet121_layers()):
    rng = np.random.default_rng([42, li])
    a = rng.standard_normal(L.m * L.n).astype(np.float32)
    w = rng.standard_normal(L.k * L.k).astype(np.float32)
    ts.append(sp.build_transform(sp.Kernel(L.k, w), sp.ConvSpec(L.m, L.n, L.k, L.s, L.p)))
    imgs.append(a)
torch.cuda.synchronize()
ys = [np.empty(t.rows, np.float32) for t in ts]
n = len(ts)
H = (C.c_void_p * n)(*[t._h for t in ts])
X = (C.c_void_p * n)(*[x.ctypes.data for x in imgs])
Y = (C.c_void_p * n)(*[y.ctypes.data for y in ys])
res = {
    "convolve_group (python API)": per_call(lambda: sp.convolve_group(ts, imgs)),
    "C call, prebuilt arrays": per_call(lambda: sp.lib.spconv_convolve_host_group(H, n, X, Y)),
}
xd = [torch.from_numpy(x).cuda() for x in imgs]
yd = [torch.empty(t.rows, device="cuda") for t in ts]
HX = (C.c_void_p * n)(*[x.data_ptr() for x in xd])
HY = (C.c_void_p * n)(*[y.data_ptr() for y in yd])
res["spmv_group device + sync (C call)"] = per_call(
    lambda: (sp.lib.spconv_spmv_group(H, n, HX, HY, None), torch.cuda.synchronize()))
tot_in = sum(x.nbytes for x in imgs)
buf = np.empty(tot_in // 4, np.float32)


def pack():
    o = 0
    for x in imgs:
        buf[o:o + x.size] = x
        o += x.size


res["numpy pack of the inputs (host memcpy)"] = per_call(pack)
for k_, v in res.items():
    print(f"{k_:45s} {v:8.1f} us")
