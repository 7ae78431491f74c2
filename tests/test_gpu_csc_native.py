"""GPU: a CSC conv transform is applied from its CSC storage (
the reference's CSC SpMV, inc/sparse.hpp:194-205, 214-258).

The handle keeps col_ptr / row_idx / vals only (no row-major copy); single
vectors and the geometries outside the band instantiations go through
csc_gather (per-output reads of the CSC storage at closed-form places), batches
of the band geometries through the CSC band check feeding the register-blocked
apply.  Outputs are compared bit for bit with the oracle's CSC scatter (fp32
fmaf: the device contract; fp64 with the reference's thread combine); storage
altered through device_ptrs is followed (the reference's scatter over the
altered arrays)."""
import numpy as np
import pytest

from helpers import CSC_BAND_KERNELS, problem

pytestmark = pytest.mark.gpu


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
    """A raw device pointer seen as a 1-D CUDA array (test access to a handle's arrays)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3}


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


def build(sp, spec, kern, layout=1):
    return sp.build_transform(sp.Kernel(spec[2], np.asarray(kern, np.float64)), sp.ConvSpec(*spec), layout=layout)


def apply(torch, sp, t, X, **opt):
    Xd = torch.from_numpy(np.ascontiguousarray(X, np.float32)).cuda()
    with sp.options(**opt):
        Y = sp.spmm(t, Xd)
    torch.cuda.synchronize()
    return Y.cpu().numpy()


def csc_want(orc, t, X):
    cp, ci, cv = t.export()
    return np.stack([orc.spmv_csc_f32_fma(t.rows, cp, ci, cv.astype(np.float32), x) for x in X])


SPECS = [(64, 64, 3, 1, 1), (300, 260, 7, 2, 3), (257, 193, 5, 3, 4), (130, 68, 3, 2, 0), (101, 76, 5, 1, 2),
         (101, 77, 5, 1, 2),
         (257, 193, 11, 1, 10), (70, 45, 1, 1, 1), (33, 29, 7, 1, 6), (96, 40, 5, 2, 1)]
BAND = {(k, s) for k in (1, 2, 3, 5, 7, 11) for s in (1, 2, 3)}


@pytest.mark.parametrize("zero", [False, True])
@pytest.mark.parametrize("spec", SPECS)
def test_csc_native_apply(sp, orc, torch_cuda, spec, zero):
    """No row-major arrays; batch 1, 2 (csc_gather) and 5 (CSC band path for the
    band geometries) bit-identical to the CSC scatter restatement."""
    m, n, k, s, p = spec
    kern, X = problem(orc, 41, m, n, k, batch=5)
    kern = kern.astype(np.float64)
    if zero:
        kern[np.random.default_rng(k * 7 + s).random(k * k) < 0.3] = 0.0
        kern[k * k // 2] = 1.5
    t = build(sp, spec, kern)
    assert t.layout == sp.Layout.CSC
    assert t.storage_bytes == 8 * t.nnz + 4 * (t.cols + 1)  # the CSC storage only
    want = csc_want(orc, t, X)
    # (the CSR ordered-fmaf chain: the same sums)
    assert np.array_equal(bits(want), bits(orc.spmm_native(*orc.build_native(*spec, kern.astype(np.float32)), X)))
    for b in (1, 2, 5):
        Y = apply(torch_cuda, sp, t, X[:b])
        assert np.array_equal(bits(Y), bits(want[:b])), (spec, b)
        if b >= 3 and (k, s) in BAND and (not zero or k <= 7):  # (zero-tap masks: k <= 7)
            assert t.last_kernel in CSC_BAND_KERNELS, t.last_kernel
        else:  # (one or two images, k <= 7: the row-at-a-time PDL form)
            assert t.last_kernel == ("csc_gather_lat" if b <= 2 and k <= 7 else "csc_gather"), t.last_kernel
    assert t.band_check_status()[1] == 0 if (k, s) in BAND else True


@pytest.mark.parametrize("fused", ["0", "1"])
@pytest.mark.parametrize("spec", [(256, 256, 3, 1, 1), (300, 260, 7, 2, 3), (130, 68, 3, 2, 0), (101, 76, 5, 1, 2)])
def test_csc_band_forms(sp, orc, torch_cuda, spec, fused):
    """Both band forms over CSC storage (separate check / fused into the apply's
    producer warp), dense and zero-tap, incl. non-finite inputs (the zero-tap
    apply redoes such outputs per entry from the staged window)."""
    m, n, k = spec[:3]
    kern, X = problem(orc, 42, m, n, k, batch=6)
    for zero in (False, True):
        kk = kern.astype(np.float64).copy()
        if zero:
            kk[1] = 0.0
        t = build(sp, spec, kk)
        Xn = X.copy()
        Xn[2, 5] = np.inf
        Xn[3, m * n // 2] = np.nan
        Y = apply(torch_cuda, sp, t, Xn, fused=fused)
        assert t.last_kernel in CSC_BAND_KERNELS
        assert np.array_equal(bits(Y), bits(csc_want(orc, t, Xn))), (spec, zero)
        segs, bad = t.band_check_status()
        seg_cols = 64 if k == 7 else 128  # (s * the check's width input columns: k7 s2 checks 32-wide)
        assert segs == m * -(-n // seg_cols) and bad == 0


@pytest.mark.slow
def test_csc_config3_full_size(sp, orc, torch_cuda):
    """BASELINE config 3 as a CSC transform: the fused CSC check + apply at the
    bench's per-GPU batches (auto form), images {0, b/2, b-1} bit-exact."""
    spec = (1024, 1024, 3, 1, 1)
    kern, X = problem(orc, 2, 1024, 1024, 3, batch=3)
    t = build(sp, spec, kern)
    cp, ci, cv = t.export()
    for batch in (96, 32):
        Xd = torch_cuda.from_numpy(np.repeat(X, (batch + 2) // 3, axis=0)[:batch]).cuda()
        Y = sp.spmm(t, Xd)
        torch_cuda.cuda.synchronize()
        assert t.last_kernel in CSC_BAND_KERNELS
        for i in (0, batch // 2, batch - 1):
            want = orc.spmv_csc_f32_fma(t.rows, cp, ci, cv.astype(np.float32), Xd[i].cpu().numpy())
            assert np.array_equal(bits(Y[i].cpu().numpy()), bits(want)), (batch, i)


@pytest.mark.parametrize("spec", [(40, 41, 5, 2, 4), (64, 64, 3, 1, 1), (17, 64, 7, 3, 0), (9, 9, 11, 1, 5)])
def test_csc_f64_thread_combine(sp, orc, ref, torch_cuda, spec):
    """spmm_f64(threads = nt) on CSC storage: the reference's per-thread partials
    over column chunks, added in thread order -- bit-identical to the compiled
    reference's spmv(m, x, nt) and to the restatement; CSR ignores nt."""
    m, n, k = spec[:3]
    rng = np.random.default_rng(k + 100)
    kern = rng.standard_normal(k * k)
    kern[rng.random(k * k) < 0.2] = 0.0
    X = rng.standard_normal((2, m * n)) * np.exp(rng.uniform(-20, 20, (2, m * n)))
    t = build(sp, spec, kern)
    tr = ref.build(*spec, kern, layout=1)
    cp, ci, cv = tr.export()
    Xd = torch_cuda.from_numpy(X).cuda()
    for nt in (1, 2, 3, 7, 16):
        Y = sp.spmm_f64(t, Xd, threads=nt).cpu().numpy()
        assert t.last_kernel == "csc_gather<f64>"
        want = tr.convolve(X, threads=nt)
        assert np.array_equal(bits64(Y), bits64(want)), nt
        for b in range(2):
            assert np.array_equal(bits64(Y[b]), bits64(orc.spmv_csc_f64_threads(t.rows, cp, ci, cv, X[b], nt)))
    # the drop-in convolve() with threads
    out = sp.convolve(t, X[0].reshape(m, n), threads=3).reshape(-1)
    assert np.array_equal(bits64(out), bits64(tr.convolve(X[:1], threads=3)[0]))
    tcsr = build(sp, spec, kern, layout=0)
    y1 = sp.spmm_f64(tcsr, Xd, threads=1).cpu().numpy()
    assert np.array_equal(bits64(sp.spmm_f64(tcsr, Xd, threads=7).cpu().numpy()), bits64(y1))


@pytest.mark.parametrize("spec", [(70, 52, 3, 1, 1), (61, 47, 5, 3, 2)])
def test_csc_storage_altered_through_device_ptrs(sp, orc, torch_cuda, spec):
    """Once device_ptrs hands the CSC arrays out, every apply first checks them
    on the device; altered storage (a value, a row index, a column's entries
    moved) is then applied as it stands -- the reference's scatter over the
    altered arrays, fp32 and fp64 -- and an untouched exposed handle still takes
    the native kernels."""
    m, n, k = spec[:3]
    kern, X = problem(orc, 43, m, n, k, batch=4)
    t = build(sp, spec, kern)
    clean = apply(torch_cuda, sp, t, X)
    cp_d, ci_d, cv_d = t.device_ptrs()
    again = apply(torch_cuda, sp, t, X)
    assert t.last_kernel != "csc_gather<verify>+csc_repair"
    assert np.array_equal(bits(again), bits(clean))
    cp, ci, cv = t.export()
    dci = torch_cuda.as_tensor(_DevArray(ci_d, t.nnz, "<i4"), device="cuda")
    dcv = torch_cuda.as_tensor(_DevArray(cv_d, t.nnz, "<f4"), device="cuda")
    e1, e2 = t.nnz // 3, (2 * t.nnz) // 3
    cv = cv.copy()
    ci = ci.copy()
    cv[e1] = np.float32(cv[e1] * 3.0)
    ci[e2] = (ci[e2] + 7 * (n // 2)) % t.rows  # an entry moved to another output row
    dcv[e1] = float(cv[e1])
    dci[e2] = int(ci[e2])
    torch_cuda.cuda.synchronize()
    Y = apply(torch_cuda, sp, t, X)
    assert t.last_kernel == "csc_gather<verify>+csc_repair"
    want = np.stack([orc.spmv_csc_f32_fma(t.rows, cp, ci, cv, x) for x in X])
    assert not np.array_equal(bits(want), bits(clean))
    assert np.array_equal(bits(Y), bits(want))
    X64 = X.astype(np.float64)
    for nt in (1, 5):
        Y64 = sp.spmm_f64(t, torch_cuda.from_numpy(X64).cuda(), threads=nt).cpu().numpy()
        w64 = np.stack([orc.spmv_csc_f64_threads(t.rows, cp, ci, cv.astype(np.float64), x, nt) for x in X64])
        assert np.array_equal(bits64(Y64), bits64(w64)), nt


def test_csc_wide_kernel_and_spgemm(sp, orc, torch_cuda):
    """k > 32 (beyond the CSC kernels) still builds a CSC handle (host
    transposition, applied through its row-major arrays); spgemm accepts CSC
    conv operands (a row-major twin for the call)."""
    spec = (40, 38, 33, 1, 16)
    rng = np.random.default_rng(3)
    kern = rng.standard_normal(33 * 33).astype(np.float32)
    t = build(sp, spec, kern)
    assert t.layout == sp.Layout.CSC
    ptr, idx, val = orc.build_transform(*spec, kern.astype(np.float64))
    want = orc.transpose(ptr.size - 1, 40 * 38, ptr, idx, val)
    assert all(np.array_equal(a, b) for a, b in zip(t.export(), want))
    X = rng.standard_normal((3, 40 * 38)).astype(np.float32)
    assert np.array_equal(bits(apply(torch_cuda, sp, t, X)), bits(orc.spmm_native(*orc.build_native(*spec, kern), X)))
    # spgemm with a CSC conv operand: T (CSC) times the identity == T
    spec2 = (20, 18, 3, 2, 1)
    k2 = rng.standard_normal(9)
    T = build(sp, spec2, k2)
    Tcsr = build(sp, spec2, k2, layout=0)
    eye = sp.Transform.from_host(T.cols, T.cols, np.arange(T.cols + 1), np.arange(T.cols), np.ones(T.cols))
    G = sp.spgemm(T, eye)
    assert all(np.array_equal(a, b) for a, b in zip(G.export(), Tcsr.export()))


@pytest.mark.parametrize("spec", [(64, 300, 7, 2, 3), (40, 290, 3, 2, 1), (50, 280, 5, 2, 2), (30, 400, 7, 3, 3),
                                  (48, 300, 11, 2, 5), (36, 390, 5, 3, 0)])
def test_csc_band_check_detects_interior_changes(sp, orc, torch_cuda, spec):
    """Exposed CSC storage of a band geometry is verified by the CSC band check
    itself; a value or a row index changed in the middle of an interior segment
    (the periodic s >= 2 verification) is caught, and the output is the
    reference's scatter over the altered arrays.  An untouched exposed handle
    passes the same check."""
    m, n, k, s, p = spec
    kern, X = problem(orc, 44, m, n, k, batch=4)
    t = build(sp, spec, kern)
    clean = apply(torch_cuda, sp, t, X)
    cp_d, ci_d, cv_d = t.device_ptrs()
    assert np.array_equal(bits(apply(torch_cuda, sp, t, X)), bits(clean))
    assert t.last_kernel != "csc_gather<verify>+csc_repair"
    assert t.band_check_status()[1] == 0
    cp, ci, cv = t.export()
    dci = torch_cuda.as_tensor(_DevArray(ci_d, t.nnz, "<i4"), device="cuda")
    dcv = torch_cuda.as_tensor(_DevArray(cv_d, t.nnz, "<f4"), device="cuda")
    a, b = m // 2, 2 * s * 64 - 3  # an input column in the middle of the second segment
    col = a * n + b
    e0, e1 = int(cp[col]), int(cp[col + 1])
    assert e1 - e0 >= 2
    for what in ("value", "row"):
        ci2, cv2 = ci.copy(), cv.copy()
        e = (e0 + e1) // 2
        if what == "value":
            cv2[e] = np.float32(cv2[e] * -2.0 + 1.0)
            dcv[e] = float(cv2[e])
        else:
            ci2[e] = (ci2[e] + 1) % t.rows
            dci[e] = int(ci2[e])
        torch_cuda.cuda.synchronize()
        Y = apply(torch_cuda, sp, t, X)
        assert t.last_kernel == "csc_gather<verify>+csc_repair", (what, t.last_kernel)
        want = np.stack([orc.spmv_csc_f32_fma(t.rows, cp, ci2, cv2, x) for x in X])
        assert np.array_equal(bits(Y), bits(want)), what
        dcv[e] = float(cv[e])
        dci[e] = int(ci[e])
        torch_cuda.cuda.synchronize()
    assert np.array_equal(bits(apply(torch_cuda, sp, t, X)), bits(clean))
    assert t.last_kernel != "csc_gather<verify>+csc_repair"
