"""Generates tests/golden/golden.npz and golden.json FROM THE REFERENCE ITSELF.

Runs the reference headers compiled unmodified into oracle/_ref/libspconv_ref.so
(``make -C oracle``; needs /root/reference, i.e. this container, not the GPU
box).  The committed outputs pin the C restatement (oracle/spconv_oracle.c) and,
through it, the device path:

* known-answer RNG values (inc/rng.hpp) and the SPEC examples;
* full CSR + fp64 outputs for config 1 (64x64 k3 s1 p1) and small cases;
* the same in CSC layout (build_transform(..., Layout::CSC)), config 1 in full;
* SHA-256 digests of the reference CSR (int64 ptr/idx, float64 val, little
  endian) and of its fp64 convolve() output for config 2 (512^2 k5 s2 p2), the
  36 config-5 edge-sweep specs on 257x193 (with the BASELINE kernel and with a
  zero-tap kernel), and a digest-of-digests over an exhaustive small sweep.

Inputs follow the SURVEY 8(d) recipe: S = derive_seed(42, cfg), kernel =
random_normal_kernel(k, derive_seed(S, 1)), image = random_normal_grid(m, n,
derive_seed(S, 2)), both rounded to fp32 so the fp32 device path sees the
same numbers.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Ref  # noqa: E402

BASE_SEED = 42


def f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).astype(a.dtype.newbyteorder("<"), copy=False).tobytes())
    return h.hexdigest()


def problem(ref: Ref, cfg: int, m: int, n: int, k: int):
    S = ref.derive_seed(BASE_SEED, cfg)
    kern = f32(ref.random_normal_kernel(k, ref.derive_seed(S, 1)))
    img = f32(ref.random_normal_grid(m, n, ref.derive_seed(S, 2)))
    return kern, img


def zero_tap_kernel(ref: Ref, k: int, seed: int):
    """Seeded kernel with roughly a third of its taps forced to +-0.0."""
    kern = f32(ref.random_normal_kernel(k, seed))
    u = ref.random_normal_grid(1, k * k, seed ^ 0x5A5A)
    kern[u > 0.45] = 0.0
    kern[u < -1.2] = -0.0
    return kern


def edge_specs():
    out = []
    for k in (1, 3, 5, 11):
        for s in (1, 2, 3):
            for p in sorted({0, 1, k - 1}):
                out.append((257, 193, k, s, p))
    return out


def sweep_specs(max_dim=9):
    for m in range(1, max_dim + 1):
        for n in range(1, max_dim + 1):
            for p in range(0, 4):
                for s in range(1, 4):
                    for k in range(1, min(m, n) + 2 * p + 1):
                        yield (m, n, k, s, p)


def main():
    ref = Ref()
    js = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj/include/spconv",
          "base_seed": BASE_SEED}
    npz = {}

    # Known-answer values (inc/rng.hpp:53-98) and Theorem 2.1 / SPEC examples.
    js["derive_seed_42_0"] = str(ref.derive_seed(42, 0))
    js["normal_42_first3"] = [float(v) for v in ref.random_normal_grid(1, 3, 42)]
    js["nnz_bound_3_3_3_1_1"] = ref.nnz_bound(3, 3, 3, 1, 1)
    js["nnz_bound_4_4_3_1_0"] = ref.nnz_bound(4, 4, 3, 1, 0)
    js["nnz_bound_1_1_1_1_2"] = ref.nnz_bound(1, 1, 1, 1, 2)
    t = ref.build(3, 3, 3, 1, 1, np.ones(9))
    js["ones_3x3_k3_p1_row_ptr"] = t.export()[0].tolist()
    js["ones_3x3_k3_p1_conv"] = t.convolve(np.ones((1, 9)))[0].tolist()
    # 4x4 input 1..16, k=2 all-ones, s=2, p=0.  The code (and
    # arithmetic) give [[14,22],[46,54]]; SPEC.md's [[14,22],[38,54]] is a typo.
    t = ref.build(4, 4, 2, 2, 0, np.ones(4))
    js["spec175_conv"] = t.convolve(np.arange(1, 17, dtype=np.float64)[None])[0].tolist()

    # Config 1 in full.
    kern, img = problem(ref, 0, 64, 64, 3)
    t = ref.build(64, 64, 3, 1, 1, kern)
    ptr, idx, val = t.export()
    y = t.convolve(img[None])[0]
    npz.update(c1_kernel=kern, c1_image=img, c1_ptr=ptr, c1_idx=idx, c1_val=val, c1_y=y)
    # ... and in CSC layout (build_transform(..., Layout::CSC)); its convolve()
    # (spmv_csc_cols, one thread) reproduces the CSR output bit for bit.
    tc = ref.build(64, 64, 3, 1, 1, kern, layout=1)
    cptr, cidx, cval = tc.export()
    yc = tc.convolve(img[None])[0]
    assert np.array_equal(yc.view(np.uint64), y.view(np.uint64))
    npz.update(c1_csc_ptr=cptr, c1_csc_idx=cidx, c1_csc_val=cval)

    # Zero-tap kernel, small: nnz(T) < Theorem 2.1 bound (SURVEY hard part 2).
    zk = np.array([1.5, 0.0, -2.0, -0.0, 3.0, 0.0, 0.25, 0.0, -1.0])
    t = ref.build(3, 3, 3, 1, 1, zk)
    ptr, idx, val = t.export()
    npz.update(zt_kernel=zk, zt_ptr=ptr, zt_idx=idx, zt_val=val)

    # Digests: config 2 and the config-5 edge sweep.
    digests = {}
    cases = [(1, (512, 512, 5, 2, 2))] + [(4, s) for s in edge_specs()]
    for cfg, (m, n, k, s, p) in cases:
        for variant in ("normal", "zerotap"):
            kern, img = problem(ref, cfg, m, n, k)
            if variant == "zerotap":
                if k == 1:
                    continue
                kern = zero_tap_kernel(ref, k, ref.derive_seed(ref.derive_seed(BASE_SEED, cfg), 99))
            t = ref.build(m, n, k, s, p, kern)
            ptr, idx, val = t.export()
            yv = t.convolve(img[None])[0]
            tc = ref.build(m, n, k, s, p, kern, layout=1)
            yc = tc.convolve(img[None])[0]
            key = f"{m}x{n}_k{k}_s{s}_p{p}_{variant}"
            digests[key] = dict(spec=[m, n, k, s, p], cfg=cfg, variant=variant, nnz=int(val.size),
                                csr=sha(ptr, idx, val), y=sha(yv), csc=sha(*tc.export()),
                                y_csc=sha(yc))
    js["digests"] = digests

    # Digest-of-digests over the exhaustive m,n <= 9 sweep (verify.hpp:66-71 grid),
    # seeded kernels as in inc/verify.hpp:47-55 (first all-non-zero draw).
    h = hashlib.sha256()
    count = 0
    for ci, (m, n, k, s, p) in enumerate(sweep_specs()):
        seed = ref.derive_seed(BASE_SEED, 1000 + ci)
        kern = f32(ref.random_normal_kernel(k, seed))
        img = f32(ref.random_normal_grid(m, n, ref.derive_seed(seed, 2)))
        t = ref.build(m, n, k, s, p, kern)
        ptr, idx, val = t.export()
        yv = t.convolve(img[None])[0]
        h.update(sha(ptr, idx, val, yv).encode())
        count += 1
    js["sweep9"] = dict(specs=count, digest=h.hexdigest())

    # Transform text (write_transform, inc/conv.hpp:221-224): digests of the
    # reference's bytes for built transforms, kernels given as fp32 bit patterns.
    text = []
    tcases = [(0, (64, 64, 3, 1, 1), "normal"), (4, (257, 193, 3, 2, 1), "normal"),
              (4, (257, 193, 5, 3, 4), "zerotap"), (4, (257, 193, 11, 1, 10), "normal"),
              (4, (257, 193, 1, 1, 1), "normal"), (6, (20, 17, 3, 1, 1), "nan")]
    for cfg, (m, n, k, s, p), variant in tcases:
        kern, _ = problem(ref, cfg, m, n, k)
        if variant == "zerotap":
            kern = zero_tap_kernel(ref, k, ref.derive_seed(ref.derive_seed(BASE_SEED, cfg), 99))
        if variant == "nan":
            kern = kern.copy()
            kern[0] = np.nan
            kern[4] = -np.nan
        t = ref.build(m, n, k, s, p, kern)
        data = t.write_text()
        data_csc = ref.build(m, n, k, s, p, kern, layout=1).write_text()
        text.append(dict(spec=[m, n, k, s, p], variant=variant,
                         kernel_bits=[int(b) for b in np.asarray(kern, np.float32).view(np.uint32)],
                         bytes=len(data), sha=hashlib.sha256(data).hexdigest(),
                         csc_bytes=len(data_csc), csc_sha=hashlib.sha256(data_csc).hexdigest()))
    js["text"] = text

    # %.17g of fp32 values widened to double, as the reference prints them
    # (format_value, inc/grid.hpp:54-59, via write_sparse of a 1 x N matrix).
    rng = np.random.default_rng(2411)
    special = np.array([0.0, -0.0, 1.0, -1.0, 0.1, 1e-4, 9.99999e-5, 1e-5, 1e16, 1e17, 9.9999998e16,
                        1.0000001e17, 123456789.0, 3.4028235e38, -3.4028235e38, 1.17549435e-38,
                        1.4e-45, -1.4e-45, 2.0 ** -126, 2.0 ** 24, 2.0 ** 57, 0.5, 0.25, 1e38, 1e-38,
                        np.inf, -np.inf, np.nan, -np.nan, 16777217.0, 1e-45 * 3, 5e-324 * 0],
                       dtype=np.float32)
    bits = np.concatenate([special.view(np.uint32),
                           rng.integers(0, 2 ** 32, 3000, dtype=np.uint64).astype(np.uint32),
                           rng.integers(0, 2 ** 23, 300, dtype=np.uint64).astype(np.uint32),  # subnormals
                           (np.float32(10.0) ** np.arange(-45, 39, dtype=np.float32)).view(np.uint32)])
    vals = bits.view(np.float32).astype(np.float64)
    N = vals.size
    data = ref.write_sparse_csr(1, N, np.array([0, N]), np.arange(N), vals).decode()
    lines = data.split("\n")[2:2 + N]
    js["g17"] = [[int(b), ln.split(" ")[2]] for b, ln in zip(bits, lines)]

    # The reference's own self-test summary (inc/verify.hpp:59-169), small grid.
    js["run_verification_6x1"] = ref.run_verification(6, 1)
    js["run_verification_12x3"] = ref.run_verification(12, 3)  # VerifyOptions defaults

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **npz)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(js, f, indent=1, sort_keys=True)
    print(f"wrote golden.npz ({len(npz)} arrays) and golden.json ({len(digests)} digests, "
          f"sweep {count} specs)")


if __name__ == "__main__":
    main()
