"""GPU: the fp64 (reference-arithmetic) apply of batches through the band path
(spconv_spmm_f64: the band check, then the register-blocked apply with the
reference's per-entry double multiply and add, inc/sparse.hpp:185-191).

Outputs are compared BIT FOR BIT with the oracle's fp64 restatement of
spmv_csr_rows over the exact stored values (fp32-representable taps and
arbitrary double taps, dense and zero-tap kernels, CSR and CSC storage), with
the fp64 thread-per-row kernel as a second witness."""
import numpy as np
import pytest

from helpers import problem

pytestmark = pytest.mark.gpu

BAND64 = ("conv_band_check+conv_spmm_band<f64>", "conv_band_check<csc>+conv_spmm_band<f64>")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture(scope="module")
def sp(torch_cuda):
    import paper_2411_19419_b200 as sp
    return sp


class _DevArray:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3}


def bits64(a):
    a = np.ascontiguousarray(a, np.float64)
    v = a.view(np.uint64).copy()
    v[np.isnan(a)] = 0x7FF8000000000000
    return v


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("spec", [(64, 64, 3, 1, 1), (130, 68, 3, 2, 0), (101, 76, 5, 1, 2), (96, 40, 5, 2, 1),
                                  (300, 260, 7, 2, 3), (257, 194, 3, 1, 0)])
def test_f64_band_bitexact(sp, orc, torch_cuda, spec, layout, opts):
    m, n, k = spec[:3]
    rng = np.random.default_rng(k * 31 + n)
    _, X32 = problem(orc, 51, m, n, k, batch=5)
    X = X32.astype(np.float64) * np.exp(rng.uniform(-3, 3, X32.shape))  # not fp32 numbers
    Xd = torch_cuda.from_numpy(X).cuda()
    for variant in ("f32taps", "f64taps", "zerotap"):
        kern = rng.standard_normal(k * k)
        if variant == "f32taps":
            kern = kern.astype(np.float32).astype(np.float64)
        if variant == "zerotap":
            kern[rng.random(k * k) < 0.3] = 0.0
            kern[k * k // 2] = 0.75
        t = sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec), layout=layout)
        Y = sp.spmm_f64(t, Xd).cpu().numpy()
        assert t.last_kernel == BAND64[layout], (variant, t.last_kernel)
        ptr, idx, val = orc.build_transform(*spec, kern)
        want = np.stack([orc.spmv_f64(ptr, idx, val, x) for x in X])
        assert np.array_equal(bits64(Y), bits64(want)), (spec, layout, variant)
        opts(path="generic")  # the thread-per-row / gather kernels agree
        Y2 = sp.spmm_f64(t, Xd).cpu().numpy()
        opts(path="auto")
        assert t.last_kernel != BAND64[layout]
        assert np.array_equal(bits64(Y2), bits64(want))


def test_f64_band_nonfinite_and_ldx(sp, orc, torch_cuda):
    """Non-finite inputs (the zero-tap apply redoes such outputs per entry),
    padded leading dimensions, batch tails."""
    spec = (70, 52, 3, 1, 1)
    rng = np.random.default_rng(9)
    kern = rng.standard_normal(9)
    kern[4] = 0.0
    t = sp.build_transform(sp.Kernel(3, kern), sp.ConvSpec(*spec))
    B, ld = 7, 70 * 52 + 6
    X = rng.standard_normal((B, ld))
    X[1, 10] = np.inf
    X[2, 500] = np.nan
    X[5, 3] = -np.inf
    Xd = torch_cuda.from_numpy(X).cuda()[:, : 70 * 52]
    Y = torch_cuda.zeros(B, t.rows + 2, dtype=torch_cuda.float64, device="cuda")[:, : t.rows]
    sp.spmm_f64(t, Xd, Y)
    assert t.last_kernel == BAND64[0]
    ptr, idx, val = orc.build_transform(*spec, kern)
    want = np.stack([orc.spmv_f64(ptr, idx, val, X[b, : 70 * 52]) for b in range(B)])
    assert np.array_equal(bits64(Y.cpu().numpy()), bits64(want))


def test_f64_band_reads_the_matrix(sp, orc, torch_cuda):
    """A CSR entry altered through device_ptrs fails its segment's check; that
    segment's rows are then summed per entry from the stored CSR (the exact
    double of the entry when the handle keeps one)."""
    spec = (128, 128, 3, 1, 1)
    rng = np.random.default_rng(4)
    kern = rng.standard_normal(9).astype(np.float32).astype(np.float64)
    t = sp.build_transform(sp.Kernel(3, kern), sp.ConvSpec(*spec))
    X = rng.standard_normal((4, 128 * 128))
    Xd = torch_cuda.from_numpy(X).cuda()
    ptr, idx, val = orc.build_transform(*spec, kern)
    _, ci, cv = t.device_ptrs()
    dcv = torch_cuda.as_tensor(_DevArray(cv, t.nnz, "<f4"), device="cuda")
    dci = torch_cuda.as_tensor(_DevArray(ci, t.nnz, "<i4"), device="cuda")
    e1, e2 = int(ptr[5000]) + 1, int(ptr[9000])
    val = val.copy()
    idx = idx.copy()
    val[e1] = np.float64(np.float32(val[e1] * 5))
    idx[e2] -= 128 * 20
    dcv[e1] = float(val[e1])
    dci[e2] = int(idx[e2])
    torch_cuda.cuda.synchronize()
    Y = sp.spmm_f64(t, Xd).cpu().numpy()
    assert t.last_kernel == BAND64[0]
    want = np.stack([orc.spmv_f64(ptr, idx, val, x) for x in X])
    assert np.array_equal(bits64(Y), bits64(want))
    assert t.band_check_status()[1] >= 1
