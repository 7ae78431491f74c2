"""One hot-path operation, run `warm` times and then once more, for an ncu
capture of the last launch(es) (gpu_round.sh).   python scripts/ncu_target.py <target> [warm]

targets: c3 (config 3, 256 images, CSR), c3b32 (32 images), c3csc (CSC storage),
c3f64 (fp64 apply), c4 (config 4, 8 images), c2 (config 2 single image),
build3 / build4 (the CSR builds), c5k11 (257 x 193, k11 s1 p10, 256 images),
group (the DenseNet121 table in one grouped launch)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402

target = sys.argv[1]
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
SPECS = {"c3": ((1024, 1024, 3, 1, 1), 256, 0), "c3b32": ((1024, 1024, 3, 1, 1), 32, 0),
         "c3csc": ((1024, 1024, 3, 1, 1), 256, 1), "c3f64": ((1024, 1024, 3, 1, 1), 256, 0),
         "c4": ((4096, 4096, 7, 2, 3), 8, 0), "c4csc": ((4096, 4096, 7, 2, 3), 8, 1), "c2": ((512, 512, 5, 2, 2), 1, 0),
         "build3": ((1024, 1024, 3, 1, 1), 0, 0), "build4": ((4096, 4096, 7, 2, 3), 0, 0),
         "c5k11": ((257, 193, 11, 1, 10), 256, 0), "k11a": ((1024, 1024, 11, 1, 5), 32, 0)}
if target == "generic3":  # config 3's matrix uploaded as a generic host CSR, 256 images
    spec = (1024, 1024, 3, 1, 1)
    t0 = sp.build_transform(sp.Kernel(3, np.random.default_rng(0).standard_normal(9).astype(np.float32)),
                            sp.ConvSpec(*spec))
    ptr, idx, val = t0.export()
    t = sp.Transform.from_host(t0.rows, t0.cols, ptr, idx, val)
    X = torch.randn(256, t.cols, device="cuda")
    Y = torch.empty(256, t.rows, device="cuda")
    for _ in range(warm + 1):
        sp.spmm(t, X, Y)
    torch.cuda.synchronize()
    print(target, t.last_kernel)
    sys.exit(0)
if target == "group":
    from paper_2411_19419_b200.layers import densenet121_layers
    ts, xs = [], []
    for li, L in enumerate(densenet121_layers()):
        rng = np.random.default_rng([42, li])
        ts.append(sp.build_transform(sp.Kernel(L.k, rng.standard_normal(L.k * L.k).astype(np.float32)),
                                     sp.ConvSpec(L.m, L.n, L.k, L.s, L.p)))
        xs.append(torch.randn(L.m * L.n, device="cuda"))
    ys = [torch.empty(t.rows, device="cuda") for t in ts]
    for _ in range(warm + 1):
        sp.spmv_group(ts, xs, ys)
    torch.cuda.synchronize()
    print(target, ts[0].last_kernel)
    sys.exit(0)
spec, b, layout = SPECS[target]
k = spec[2]
kern = sp.Kernel(k, np.random.default_rng(0).standard_normal(k * k).astype(np.float32))
if b == 0:
    for _ in range(warm + 1):
        t = sp.build_transform(kern, sp.ConvSpec(*spec))
        torch.cuda.synchronize()
        t.close()
    sys.exit(0)
t = sp.build_transform(kern, sp.ConvSpec(*spec), layout=layout)
dt = torch.float64 if target == "c3f64" else torch.float32
X = torch.randn(b, t.cols, device="cuda", dtype=dt)
Y = torch.empty(b, t.rows, device="cuda", dtype=dt)
fn = (lambda: sp.spmm_f64(t, X, Y)) if dt == torch.float64 else (lambda: sp.spmm(t, X, Y))
for _ in range(warm + 1):
    fn()
torch.cuda.synchronize()
print(target, t.last_kernel)
