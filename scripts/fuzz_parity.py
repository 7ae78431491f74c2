#!/usr/bin/env python
"""Randomised GPU parity fuzzing (a long-running complement to tests/):
random geometries (m, n up to 300, k up to 11, s up to 4, p up to k), dense /
zero-tap / non-finite kernels and the reference's own double taps (exact
fp64 values: export and the fp64 apply checked bit for bit), every build
kernel, CSR and CSC layouts, batches 1-9 through the
default path and every forced path, padded ldx, the fused and two-kernel band
forms; every output compared BIT-EXACTLY with the oracle's ordered-fmaf
restatement and every matrix with the oracle's build.

    python scripts/fuzz_parity.py SECONDS [SEED] > report.txt
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_19419_b200 as sp  # noqa: E402
from oracle import Oracle  # noqa: E402

PATHS = [None, "spmv", "spmv_plain", "banded", "tiled", "tiled_notma", "generic"]


def bits64(a):
    a = np.ascontiguousarray(a, np.float64)
    v = a.view(np.uint64).copy()
    v[np.isnan(a)] = 0x7FF8000000000000
    return v


def bits(a):
    a = np.ascontiguousarray(a, np.float32)
    v = a.view(np.uint32).copy()
    v[np.isnan(a)] = 0x7FC00000
    return v


def main():
    secs = float(sys.argv[1])
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rng = np.random.default_rng(seed)
    orc = Oracle()
    t_end = time.time() + secs
    cases = fails = groups = 0
    pending, group_at = [], 8
    while time.time() < t_end:
        k = int(rng.choice([1, 2, 3, 3, 3, 5, 5, 7, 7, 11]))
        s = int(rng.choice([1, 1, 2, 2, 3, 4]))
        p = int(rng.integers(0, k + 1))
        m = int(rng.integers(max(1, k - 2 * p), 300))
        n = int(rng.choice([int(rng.integers(max(1, k - 2 * p), 300)), 4 * int(rng.integers(1, 70))]))
        if orc.spec_check(m, n, k, s, p):
            continue
        kern64 = rng.standard_normal(k * k)  # mode 2: the reference's own double taps
        kern = kern64.astype(np.float32)
        mode = rng.integers(0, 10)
        if mode == 0:
            kern[rng.random(k * k) < 0.3] = 0.0
        elif mode == 1:
            kern[rng.integers(0, k * k)] = np.nan
        if mode != 2:
            kern64 = kern.astype(np.float64)
        batch = int(rng.integers(1, 10))
        X = rng.standard_normal((batch, m * n)).astype(np.float32)
        if rng.random() < 0.1:
            X[0, rng.integers(0, m * n)] = np.inf
        layout = sp.Layout.CSC if rng.random() < 0.25 else sp.Layout.CSR
        spec = sp.ConvSpec(m, n, k, s, p)
        build = str(rng.choice(["auto", "auto", "block", "warp", "persist"]))
        with sp.options(build=build):
            t = sp.build_transform(sp.Kernel(k, kern64), spec, layout=layout)
        rp, ri, rv = orc.build_native(m, n, k, s, p, kern)
        ptr = np.empty(t.rows + 1, np.int32)
        idx = np.empty(max(t.nnz, 1), np.int32)
        val = np.empty(max(t.nnz, 1), np.float32)
        p64, i64, v64 = orc.build_transform(m, n, k, s, p, kern64)  # exact doubles
        if layout == sp.Layout.CSR:
            t.copy_native(ptr, idx, val)  # the fp32 arrays the kernels read
            ok = np.array_equal(ptr, rp) and np.array_equal(idx[:t.nnz], ri) and np.array_equal(
                bits(val[:t.nnz]), bits(rv))
            wp, wi, wv = p64, i64, v64
        else:
            wp, wi, wv = orc.transpose(t.rows, t.cols, p64, i64, v64)
        gp, gi, gv = t.export()
        nz = int(wp[-1])
        ok = ok if layout == sp.Layout.CSR else True
        ok = ok and np.array_equal(gp, wp) and np.array_equal(gi[:nz], wi) and np.array_equal(
            np.nan_to_num(gv[:nz], nan=7.0).view(np.uint64), np.nan_to_num(wv, nan=7.0).view(np.uint64))
        if ok:  # fp64 apply (exact values; the band path for batches; CSC with a random thread count)
            X64 = X.astype(np.float64) * (1.0 + 2.0 ** -30)
            nt = int(rng.choice([1, 1, 2, 3, 8])) if layout == sp.Layout.CSC else 1
            y64 = sp.spmm_f64(t, torch.from_numpy(X64).cuda(), threads=nt).cpu().numpy()
            for b in range(batch):
                w64 = (orc.spmv_csc_f64_threads(t.rows, wp, wi, wv, X64[b], nt) if layout == sp.Layout.CSC
                       else orc.spmv_f64(p64, i64, v64, X64[b]))
                ok = ok and np.array_equal(bits64(y64[b]), bits64(w64))
        want = orc.spmm_native(rp, ri, rv, X)
        pad = int(rng.choice([0, 0, 4]))
        Xd = torch.zeros(batch, m * n + pad, device="cuda")
        Xd[:, :m * n] = torch.from_numpy(X)
        path = PATHS[int(rng.integers(0, len(PATHS)))] if rng.random() < 0.4 else None
        env = {}
        if path:
            env["path"] = path
        if rng.random() < 0.3:
            env["fused"] = str(int(rng.integers(0, 2)))
        if rng.random() < 0.3:
            env["stage"] = str(rng.choice(["bulk", "window"]))
        try:
            with sp.options(**env):
                Y = sp.spmm(t, Xd[:, :m * n])
            torch.cuda.synchronize()
            got = Y.cpu().numpy()
            ok_y = np.array_equal(bits(got), bits(want))
        except (ValueError, RuntimeError) as e:  # a forced path may not support the geometry
            ok_y = path is not None and ("unsupported" in str(e) or "longer than" in str(e))
            if not ok_y:
                print("ERROR", (m, n, k, s, p), batch, env, e)
        cases += 1
        if not (ok and ok_y):
            fails += 1
            print("FAIL", (m, n, k, s, p), "mode", int(mode), "build", build, "batch", batch, "layout", layout, "env", env,
                  "matrix_ok", ok, "y_ok", ok_y, "kernel", t.last_kernel, flush=True)
        # every few cases the transform joins a pending group; groups of 2..40
        # members are applied in one call (fp32 device / host, fp64 host) and
        # each member compared with its own oracle output
        if rng.random() < 0.3:
            x0 = X[0].copy()
            x64 = x0.astype(np.float64) * (1.0 + 2.0 ** -30)
            pending.append((t, x0, want[0].copy(), x64, orc.spmv_f64(p64, i64, v64, x64)))
            t = None
        if len(pending) >= group_at:
            gts = [q[0] for q in pending]
            ys = sp.spmv_group(gts, [torch.from_numpy(q[1]).cuda() for q in pending])
            torch.cuda.synchronize()
            yh = sp.convolve_group(gts, [q[1] for q in pending])
            y64 = sp.convolve_group_f64(gts, [q[3] for q in pending])
            for q, a, b, c in zip(pending, ys, yh, y64):
                if not (np.array_equal(bits(a.cpu().numpy()), bits(q[2])) and np.array_equal(bits(b), bits(q[2]))
                        and np.array_equal(bits64(c), bits64(q[4]))):
                    fails += 1
                    print("FAIL group member", q[0].spec, q[0].layout, flush=True)
            groups += 1
            for q in pending:
                q[0].close()
            pending.clear()
            group_at = int(rng.integers(2, 41))
        if t is not None:
            t.close()
    print(f"fuzz: {cases} cases, {groups} groups, {fails} failures (seed {seed}, {secs:.0f} s)")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
