"""Shared test helpers: the SURVEY 8(d) seeded problems (via the oracle's
restated RNG), digest helpers matching tests/golden/make_golden.py, spec lists."""
from __future__ import annotations

import hashlib

import numpy as np

BASE_SEED = 42

# BASELINE.json configs (index = cfg used in derive_seed(42, cfg)).
CONFIGS = {
    0: (64, 64, 3, 1, 1),
    1: (512, 512, 5, 2, 2),
    2: (1024, 1024, 3, 1, 1),
    3: (4096, 4096, 7, 2, 3),
}


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).astype(a.dtype.newbyteorder("<"), copy=False).tobytes())
    return h.hexdigest()


def problem(orc, cfg: int, m: int, n: int, k: int, batch: int = 1):
    """(kernel f32 [k*k], images f32 [batch, m*n]); image b uses derive_seed(S, 2+b)."""
    S = orc.derive_seed(BASE_SEED, cfg)
    kern = orc.random_normal_f32(orc.derive_seed(S, 1), k * k)
    X = np.stack([orc.random_normal_f32(orc.derive_seed(S, 2 + b), m * n) for b in range(batch)])
    return kern, X


def zero_tap_kernel(orc, k: int, seed: int) -> np.ndarray:
    """Same construction as make_golden.zero_tap_kernel, via the restated RNG."""
    kern = orc.random_normal_f32(seed, k * k).astype(np.float64)
    u = orc.random_normal(seed ^ 0x5A5A, k * k)
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


def golden_cases(orc, js):
    """Yield (key, spec, kernel f64, image f64) for every digest in golden.json."""
    for key, d in js["digests"].items():
        m, n, k, s, p = d["spec"]
        kern, X = problem(orc, d["cfg"], m, n, k)
        kern = kern.astype(np.float64)
        if d["variant"] == "zerotap":
            kern = zero_tap_kernel(orc, k, orc.derive_seed(orc.derive_seed(BASE_SEED, d["cfg"]), 99))
        yield key, (m, n, k, s, p), kern, X[0].astype(np.float64)


# Kernel pairs of the band path (spconv_csr_last_kernel): the check kernel +
# apply, or the fused check-and-apply + its fixup pass.
# (the fixup pass only once the storage was handed out by device_ptrs)
BAND_KERNELS = ("conv_band_check+conv_spmm_band", "conv_spmm_band<fused>", "conv_spmm_band<fused>+conv_band_fixup")
# ... and over CSC storage (the CSC band check; no fixup pass)
CSC_BAND_KERNELS = ("conv_band_check<csc>+conv_spmm_band", "conv_spmm_band<fused,csc>")

# The latency SpMV of conv transforms (batch <= 2): one round trip with the
# input window staged beside the matrix run, or the bulk-staged kernel
# (options stage=window / bulk; auto picks by matrix size and eligibility).
LATENCY_SPEC = ("conv_spmv_win", "csr_spmv_bulk<spec>")
