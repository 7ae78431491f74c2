"""Write-only bandwidth on this B200 for the build's roofline context: event-timed
cudaMemsetAsync and a torch fill of 80 MB (config 3's CSR) and 1.66 GB (config 4's),
L2 scrubbed before every rep.  (The build kernels themselves are event-timed by
bench.py / scripts/build_ab.py.)"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp  # noqa: E402

scrub = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=20):
    fn()
    ts = []
    for _ in range(reps):
        scrub.zero_()
        torch.cuda._sleep(200_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for name, spec in (("c3", (1024, 1024, 3, 1, 1)), ("c4", (4096, 4096, 7, 2, 3))):
    k = spec[2]
    kern = sp.Kernel(k, np.random.default_rng(0).standard_normal(k * k).astype(np.float32))
    t = sp.build_transform(kern, sp.ConvSpec(*spec))
    nbytes = 8 * t.nnz + 4 * (t.rows + 1)
    t.close()
    buf = torch.empty(nbytes // 4 + 1, dtype=torch.int32, device="cuda")
    us_memset = timed(lambda: buf.zero_())
    us_fill = timed(lambda: buf.fill_(7))
    print(f"{name}: {nbytes / 1e6:.1f} MB  memset {us_memset:.1f} us ({nbytes / us_memset / 1e3:.0f} GB/s)  "
          f"fill {us_fill:.1f} us ({nbytes / us_fill / 1e3:.0f} GB/s)", flush=True)
