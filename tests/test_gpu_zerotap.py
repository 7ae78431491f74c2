"""GPU: kernels with exact-zero taps on the band path (the ZT instantiations).

The reference drops zero taps from T (inc/sparse.hpp:335), so every row's
stored taps are a tap-mask-dependent subset of its window.  The band check
verifies that masked footprint, the blocked apply sums all k*k taps (exact for
finite inputs: fmaf(0, x, acc) == acc) and a thread that saw a non-finite sum
redoes its outputs per entry.  Outputs must equal the oracle's ordered-fmaf
restatement over the STORED entries bit for bit -- with inf / NaN inputs
placed under zero taps -- on the two-kernel and the fused forms, and a
tampered matrix must still be honoured."""
import numpy as np
import pytest

from test_gpu_parity import _DevArray, bits, build, native_copy, run_spmm
from helpers import LATENCY_SPEC, BAND_KERNELS, problem

pytestmark = pytest.mark.gpu

SPECS = [(130, 140, 3, 1, 1), (97, 92, 5, 1, 2), (120, 132, 3, 2, 1), (101, 76, 5, 2, 2), (150, 160, 7, 2, 3)]  # n % 4 == 0: TMA-able rows


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture(scope="module")
def sp(torch_cuda):
    import paper_2411_19419_b200 as sp
    return sp


def zero_kernel(rng, k, frac):
    kern = rng.standard_normal(k * k).astype(np.float32)
    z = rng.random(k * k) < frac
    z[rng.integers(0, k * k)] = False  # at least one stored tap
    kern[z] = 0.0
    kern[np.flatnonzero(z)[::2]] = -0.0  # both signed zeros are dropped
    return kern


@pytest.mark.parametrize("fused", ["0", "1"])
@pytest.mark.parametrize("spec", SPECS)
def test_zero_tap_band_bitexact(sp, orc, torch_cuda, spec, fused, opts):
    opts(fused=fused)
    m, n, k = spec[:3]
    rng = np.random.default_rng(hash(spec) % 1000)
    for frac in (0.2, 0.5, 0.8):
        kern = zero_kernel(rng, k, frac)
        _, X = problem(orc, 17, m, n, k, batch=5)
        # non-finite inputs, some under zero taps of interior outputs
        X[1, (m // 2) * n + n // 2] = np.inf
        X[2, (m // 3) * n + 7] = -np.inf
        X[3, rng.integers(0, m * n, 4)] = np.nan
        t = build(sp, spec, kern)
        ptr, idx, val = native_copy(t)
        Y = run_spmm(torch_cuda, sp, t, X)
        assert t.last_kernel in BAND_KERNELS, t.last_kernel
        segs, failed = t.band_check_status()
        assert segs > 0 and failed == 0, (spec, frac, failed)  # the masked footprint matched everywhere
        want = orc.spmm_native(ptr, idx, val, X)
        assert np.array_equal(bits(Y), bits(want)), (spec, frac)


@pytest.mark.parametrize("fused", ["0", "1"])
def test_zero_tap_band_check_reads_the_matrix(sp, orc, torch_cuda, fused, opts):
    opts(fused=fused)
    spec = (256, 256, 3, 1, 1)
    m, n, k = spec[:3]
    kern = np.array([0.5, 0.0, -1.25, 0.0, 2.0, 0.0, 0.75, 0.0, -0.5], np.float32)
    _, X = problem(orc, 18, m, n, k, batch=6)
    t = build(sp, spec, kern)
    ptr, idx, val = native_copy(t)
    clean = run_spmm(torch_cuda, sp, t, X)
    assert np.array_equal(bits(clean), bits(orc.spmm_native(ptr, idx, val, X)))
    _, ci, cv = t.device_ptrs()
    dci = torch_cuda.as_tensor(_DevArray(ci, t.nnz, "<i4"), device="cuda")
    dcv = torch_cuda.as_tensor(_DevArray(cv, t.nnz, "<f4"), device="cuda")
    r1, r2 = t.rows // 2 + 100, t.rows // 3 + 17
    e_col, e_val = int(ptr[r1]) + 1, int(ptr[r2 + 1]) - 1
    idx[e_col] += 1  # a dropped (zero-tap) column now stored
    val[e_val] = np.float32(val[e_val] * 3.0)
    dci[e_col] = int(idx[e_col])
    dcv[e_val] = float(val[e_val])
    torch_cuda.cuda.synchronize()
    Y = run_spmm(torch_cuda, sp, t, X)
    assert t.last_kernel in BAND_KERNELS
    assert 1 <= t.band_check_status()[1] <= 2  # exactly the tampered segments failed
    want = orc.spmm_native(ptr, idx, val, X)
    assert not np.array_equal(bits(want), bits(clean))
    assert np.array_equal(bits(Y), bits(want))


@pytest.mark.parametrize("spec", SPECS + [(64, 64, 4, 3, 2)])
def test_zero_tap_latency_spmv_closed_form(sp, orc, torch_cuda, spec):
    """Batch <= 2: the latency SpMV predicts each warp's run from the tap mask
    (W[j] and the stored-tap column counts) and fetches it with no dependent
    row_ptr load; bit-exact, including the prediction-mismatch path
    (option spec_skew)."""
    import os
    m, n, k = spec[:3]
    rng = np.random.default_rng(k + 100)
    kern = zero_kernel(rng, k, 0.4)
    _, X = problem(orc, 19, m, n, k, batch=2)
    t = build(sp, spec, kern)
    ptr, idx, val = native_copy(t)
    want = orc.spmm_native(ptr, idx, val, X)
    for b in (1, 2):
        Y = run_spmm(torch_cuda, sp, t, X[:b])
        assert t.last_kernel in LATENCY_SPEC
        assert np.array_equal(bits(Y), bits(want[:b])), (spec, b)
    with sp.options(spec_skew=4):
        Y = run_spmm(torch_cuda, sp, t, X[:1])
    assert np.array_equal(bits(Y), bits(want[:1]))
