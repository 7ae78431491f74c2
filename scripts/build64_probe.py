"""Event-timed builds with fp32-exact taps against the reference's own doubles
(spconv_build_transform_f64 tag build + retag pass)."""
import statistics, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2411_19419_b200 as sp
st = torch.cuda.Stream()
for name, spec in (("c3", (1024, 1024, 3, 1, 1)), ("c4", (4096, 4096, 7, 2, 3))):
    k = spec[2]
    k64 = np.random.default_rng(0).standard_normal(k * k)
    for label, taps in (("fp32 taps", k64.astype(np.float32).astype(np.float64)), ("double taps", k64)):
        ts = []
        for i in range(13):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                torch.cuda._sleep(2_000_000)
                e0.record(st)
                t = sp.build_transform(sp.Kernel(k, taps), sp.ConvSpec(*spec), stream=st)
                e1.record(st)
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
            t.close()
        print(f"{name} {label:12s} {statistics.median(ts):9.1f} us")
