"""GPU: the band path over every instantiated geometry -- k in {1, 2, 3, 5, 7, 11},
s in {1, 2, 3} -- with TMA windows (16-byte row pitch) and with cp.async
element staging (odd widths: BASELINE config 5's 257 x 193), CSR and CSC
storage, dense and zero-tap kernels, both check forms, fp32 and fp64.

Every output is compared BIT FOR BIT with the oracle's ordered restatements
(fp32 fmaf; fp64 multiply then add) of the same transform."""
import numpy as np
import pytest

from helpers import BAND_KERNELS, CSC_BAND_KERNELS, problem

pytestmark = pytest.mark.gpu

KS = [(k, s) for k in (1, 2, 3, 5, 7, 11) for s in (1, 2, 3)]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture(scope="module")
def sp(torch_cuda):
    import paper_2411_19419_b200 as sp
    return sp


def bits(a):
    a = np.ascontiguousarray(a, np.float32)
    v = a.view(np.uint32).copy()
    v[np.isnan(a)] = 0x7FC00000
    return v


def bits64(a):
    a = np.ascontiguousarray(a, np.float64)
    v = a.view(np.uint64).copy()
    v[np.isnan(a)] = 0x7FF8000000000000
    return v


@pytest.mark.parametrize("n", [196, 193])
@pytest.mark.parametrize("ks", KS)
def test_band_geometry(sp, orc, torch_cuda, ks, n, opts):
    k, s = ks
    p = [0, 1, k - 1][(k + s) % 3]
    spec = (131, n, k, s, p)
    m = 131
    kern, X = problem(orc, 61, m, n, k, batch=4)
    X = X.copy()
    X[1, 7] = np.inf  # non-finite inputs (zero-tap kernels redo such outputs per entry)
    for zero in (False, True):
        kv = kern.astype(np.float64).copy()
        if zero:
            kv[np.random.default_rng(k * 3 + s).random(k * k) < 0.3] = 0.0
            kv[(k * k) // 2] = 1.25
        want = orc.spmm_native(*orc.build_native(*spec, kv.astype(np.float32)), X)
        for layout in (0, 1):
            t = sp.build_transform(sp.Kernel(k, kv), sp.ConvSpec(*spec), layout=layout)
            for fused in ("0", "1"):
                opts(fused=fused)
                Xd = torch_cuda.from_numpy(X).cuda()
                Y = sp.spmm(t, Xd).cpu().numpy()
                banded = not (zero and k == 11)
                if banded:
                    assert t.last_kernel in BAND_KERNELS + CSC_BAND_KERNELS, (spec, layout, t.last_kernel)
                assert np.array_equal(bits(Y), bits(want)), (spec, zero, layout, fused, t.last_kernel)
            if layout == 0 and not zero:
                X64 = X.astype(np.float64) * 1.000001
                Y64 = sp.spmm_f64(t, torch_cuda.from_numpy(X64).cuda()).cpu().numpy()
                ptr, idx, val = orc.build_transform(*spec, kv)
                w64 = np.stack([orc.spmv_f64(ptr, idx, val, x) for x in X64])
                assert np.array_equal(bits64(Y64), bits64(w64)), (spec, t.last_kernel)
            if layout == 0 and banded:
                segs, bad = t.band_check_status()
                assert bad == 0


def test_band_k11_reads_the_matrix(sp, orc, torch_cuda):
    """k = 11 checks segments of 32 output columns (121 entries per row): an
    altered entry fails exactly its segment, whose rows are then summed per entry."""
    spec = (96, 200, 11, 1, 5)
    kern, X = problem(orc, 62, 96, 200, 11, batch=3)
    t = sp.build_transform(sp.Kernel(11, kern.astype(np.float64)), sp.ConvSpec(*spec))

    class _Dev:
        def __init__(self, ptr, n, ts):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": ts, "data": (ptr, False), "version": 3}

    ptr, idx, val = [np.asarray(a) for a in orc.build_native(*spec, kern)]
    _, _, cv = t.device_ptrs()
    dcv = torch_cuda.as_tensor(_Dev(cv, t.nnz, "<f4"), device="cuda")
    e = int(ptr[40 * t.spec.n_out + 77]) + 60
    val = val.copy()
    val[e] = np.float32(val[e] * -2)
    dcv[e] = float(val[e])
    torch_cuda.cuda.synchronize()
    Y = sp.spmm(t, torch_cuda.from_numpy(X).cuda()).cpu().numpy()
    assert np.array_equal(bits(Y), bits(orc.spmm_native(ptr, idx, val, X)))
    assert t.band_check_status()[1] == 1


@pytest.mark.parametrize("ks", [(3, 1), (3, 2), (5, 3), (7, 1), (11, 1), (2, 2)])
def test_odd_width_repitch_and_element_staging(sp, orc, torch_cuda, ks, opts):
    """Rows not 16-byte pitched: the default path copies the images into
    16-byte pitched rows and loads TMA windows from the copy; option
    repitch = off stages them with cp.async element copies.  Both bit-equal to
    the oracle, also with a misaligned base and a padded leading dimension,
    fp32 and fp64."""
    k, s = ks
    p = k // 2
    spec = (67, 193, k, s, p)
    kern, X = problem(orc, 63, 67, 193, k, batch=5)
    t = sp.build_transform(sp.Kernel(k, kern.astype(np.float64)), sp.ConvSpec(*spec))
    want = orc.spmm_native(*orc.build_native(*spec, kern.astype(np.float32)), X)
    ptr, idx, val = orc.build_transform(*spec, kern.astype(np.float64))
    X64 = X.astype(np.float64) * 1.000001
    w64 = np.stack([orc.spmv_f64(ptr, idx, val, x) for x in X64])
    ld = t.cols + 3
    for rp in ("auto", "off"):
        opts(repitch=rp)
        for off in (0, 1):  # (1: base 4 bytes past a 16-byte boundary)
            buf = torch_cuda.zeros(off + 5 * ld, device="cuda")
            Xd = buf[off:].view(5, ld)[:, : t.cols]
            Xd.copy_(torch_cuda.from_numpy(X))
            Y = sp.spmm(t, Xd).cpu().numpy()
            assert t.last_kernel in BAND_KERNELS, t.last_kernel
            assert np.array_equal(bits(Y), bits(want)), (ks, rp, off)
            buf64 = torch_cuda.zeros(off + 5 * ld, dtype=torch_cuda.float64, device="cuda")
            Xd64 = buf64[off:].view(5, ld)[:, : t.cols]
            Xd64.copy_(torch_cuda.from_numpy(X64))
            Y64 = sp.spmm_f64(t, Xd64).cpu().numpy()
            assert np.array_equal(bits64(Y64), bits64(w64)), (ks, rp, off, t.last_kernel)
