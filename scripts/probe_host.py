"""Host-path latency anatomy (one 56^2 k3 layer, one image): per-call wall time
of the C-ABI host call with page-locked and pageable buffers, against a bare
device-buffer SpMV + synchronize and an empty stream synchronize."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402


def per_call(fn, n=2000):
    for _ in range(50):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


for spec in ((56, 56, 3, 1, 1), (7, 7, 3, 1, 1), (224, 224, 7, 2, 3)):
    m, n, k, s, p = spec
    t = sp.build_transform(sp.Kernel(k, np.random.default_rng(0).standard_normal(k * k).astype(np.float32)),
                           sp.ConvSpec(*spec))
    xp = torch.randn(1, t.cols).pin_memory()
    yp = torch.empty(1, t.rows).pin_memory()
    xq = xp.numpy().copy()
    yq = np.empty((1, t.rows), np.float32)
    xd = xp.cuda()
    yd = torch.empty(1, t.rows, device="cuda")
    st = torch.cuda.current_stream()
    h = t._h
    L = sp.lib
    res = {
        "pinned": per_call(lambda: L.spconv_convolve_host(h, xp.data_ptr(), yp.data_ptr(), 1)),
        "pageable": per_call(lambda: L.spconv_convolve_host(h, xq.ctypes.data, yq.ctypes.data, 1)),
        "device+sync": per_call(lambda: (L.spconv_spmv(h, xd.data_ptr(), yd.data_ptr(), None), torch.cuda.synchronize())),
        "sync only": per_call(lambda: torch.cuda.synchronize()),
    }
    sp.convolve_batch(t, xp, yp)
    print(spec, t.last_kernel, {a: round(b, 2) for a, b in res.items()}, flush=True)
