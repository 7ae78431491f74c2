"""GPU: transforms of the reference's own tap type -- arbitrary doubles, as
random_normal_kernel (inc/rng.hpp) produces them -- are exact.

spconv_build_transform_f64 keeps an entry wherever the DOUBLE tap is non-zero
(inc/sparse.hpp:335) and, when some tap is not an fp32 number, the exact fp64
value of every entry.  Against the compiled reference, bit for bit:
  * export (ptr / idx / val, both layouts) == Transform::matrix storage;
  * write_transform text == the reference's file, byte for byte;
  * spmm_f64 / the drop-in convolve == the reference's convolve (fp64);
  * relayout and read_transform keep the exact values;
  * generic host matrices (read_sparse, from_host) keep theirs.
The fp32 kernels apply the narrowed taps under their own contract (compared
with the oracle's fp32 restatement on the narrowed taps)."""
import numpy as np
import pytest

from helpers import BAND_KERNELS

pytestmark = pytest.mark.gpu

SPECS = [(64, 64, 3, 1, 1), (57, 43, 5, 2, 2), (31, 40, 7, 2, 3), (20, 9, 4, 3, 2), (16, 16, 1, 1, 0)]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture(scope="module")
def sp(torch_cuda):
    import paper_2411_19419_b200 as sp
    return sp


def u64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def kernel64(ref, k, seed, zeros=False, tiny=False):
    kern = ref.random_normal_kernel(k, seed)  # the reference's doubles
    if zeros and k > 1:
        kern[1] = 0.0
        kern[-1] = -0.0
    if tiny and k > 1:
        kern[0] = 1e-300  # non-zero double, fp32 zero: the reference keeps the entry
    return kern


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("layout", [0, 1])
def test_storage_and_text_bitexact_vs_reference(sp, ref, spec, layout):
    k = spec[2]
    for variant, kw in (("normal", {}), ("zeros", {"zeros": True}), ("tiny", {"tiny": True})):
        kern = kernel64(ref, k, 7 + k, **kw)
        rt = ref.build(*spec, kern, layout=layout)
        t = sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec), layout=layout)
        assert t.layout == layout
        gp, gi, gv = t.export()
        wp, wi, wv = rt.export()
        nnz = wp[-1]
        assert np.array_equal(gp, wp), (spec, variant)
        assert np.array_equal(gi[:nnz], wi), (spec, variant)
        assert np.array_equal(u64(gv[:nnz]), u64(wv)), (spec, variant)
        assert t.write_text() == rt.write_text(), (spec, variant)


@pytest.mark.parametrize("spec", SPECS)
def test_fp64_apply_bitexact_vs_reference_convolve(sp, ref, torch_cuda, spec):
    torch = torch_cuda
    m, n, k = spec[:3]
    kern = kernel64(ref, k, 11, zeros=True, tiny=True)
    X = np.stack([ref.random_normal_grid(m, n, 100 + b).reshape(-1) for b in range(3)])
    want = ref.build(*spec, kern).convolve(X)
    for layout in (0, 1):
        t = sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec), layout=layout)
        Y = sp.spmm_f64(t, torch.from_numpy(X).cuda())
        assert np.array_equal(u64(Y.cpu().numpy()), u64(want)), (spec, layout)
        # the host-buffer fp64 path (drop-in convolve)
        Yh = np.empty_like(want)
        sp._check(sp.lib.spconv_convolve_host_f64(t._h, X.ctypes.data, Yh.ctypes.data, 3))
        assert np.array_equal(u64(Yh), u64(want))


def test_fp32_kernels_apply_narrowed_taps(sp, ref, orc, torch_cuda):
    """The fp32 SpMM (band path included) == the oracle's fp32 ordered-fmaf
    restatement on the fp32-narrowed taps."""
    torch = torch_cuda
    spec = (96, 80, 3, 1, 1)
    kern = kernel64(ref, 3, 5)
    t = sp.build_transform(sp.Kernel(3, kern), sp.ConvSpec(*spec))
    X = np.random.default_rng(3).standard_normal((8, 96 * 80)).astype(np.float32)
    Y = sp.spmm(t, torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    assert t.last_kernel in BAND_KERNELS
    want = orc.spmm_native(*orc.build_native(*spec, kern.astype(np.float32)), X)
    assert np.array_equal(Y.cpu().numpy().view(np.uint32), want.view(np.uint32))
    # a non-zero double tap that narrows to 0.0f: stored (as the reference
    # stores it) and applied as w = 0 by the masked band path
    kern2 = kernel64(ref, 3, 5, tiny=True)
    t2 = sp.build_transform(sp.Kernel(3, kern2), sp.ConvSpec(*spec))
    X[2, 500] = np.inf  # under the stored zero tap too
    Y2 = sp.spmm(t2, torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    assert t2.last_kernel in BAND_KERNELS
    ptr, idx, val = t2.export()
    want2 = orc.spmm_f32_fma(ptr, idx, val.astype(np.float32), X)
    got2 = Y2.cpu().numpy()
    assert np.isnan(want2).any()  # 0 * inf under the stored zero tap
    assert np.array_equal(np.isnan(got2), np.isnan(want2))  # (NaN payloads are not part of the contract)
    assert np.array_equal(np.nan_to_num(got2, nan=7.0).view(np.uint32), np.nan_to_num(want2, nan=7.0).view(np.uint32))


def test_relayout_and_read_keep_exact_values(sp, ref, torch_cuda):
    spec = (45, 38, 5, 2, 1)
    kern = kernel64(ref, 5, 21)  # (no zero taps: the read-back handle takes the conv kernels)
    t = sp.build_transform(sp.Kernel(5, kern), sp.ConvSpec(*spec))
    rt = ref.build(*spec, kern)
    c = sp.relayout(t, sp.Layout.CSC)
    rc = rt.relayout(1)
    (gp, gi, gv), (wp, wi, wv) = c.export(), rc.export()
    nnz = wp[-1]
    assert np.array_equal(gp, wp) and np.array_equal(gi[:nnz], wi)
    assert np.array_equal(u64(gv[:nnz]), u64(wv))
    back = sp.relayout(c, sp.Layout.CSR)
    assert back.write_text() == rt.write_text()
    # read_transform of the reference's file: adopted as a conv handle, exact
    for r_t, data in ((rt, rt.write_text()), (rc, rc.write_text())):
        r = sp.read_transform(data)
        assert r.write_text() == data
        X = torch_cuda.from_numpy(np.ones((4, 45 * 38), np.float32)).cuda()
        sp.spmm(r, X)
        torch_cuda.cuda.synchronize()
        assert r.last_kernel.startswith(("conv_", "csc_gather")), r.last_kernel  # adopted: conv kernels apply


def test_generic_host_matrix_keeps_exact_values(sp, ref, torch_cuda):
    """read_sparse / from_host of arbitrary doubles: export, text and the
    fp64 apply are exact (the reference's write_sparse / spmv)."""
    rng = np.random.default_rng(9)
    rows, cols = 37, 53
    dense = rng.standard_normal((rows, cols)) * (rng.random((rows, cols)) < 0.2)
    dense[0, 0] = 1e-310  # subnormal double
    dense[1, 2] = 3.0e300
    ptr = np.concatenate([[0], np.cumsum((dense != 0).sum(1))]).astype(np.int64)
    idx = np.nonzero(dense)[1].astype(np.int64)
    val = dense[dense != 0]
    want_text = ref.write_sparse_csr(rows, cols, ptr, idx, val)
    for layout in (0, 1):
        h = sp.Transform.from_host(rows, cols, ptr, idx, val) if layout == 0 else \
            sp.Transform.from_host(rows, cols, *_csc(rows, cols, ptr, idx, val), layout=1)
        if layout == 0:
            assert h.write_text(transform_header=False) == want_text
            gp, gi, gv = h.export()
            assert np.array_equal(u64(gv[:val.size]), u64(val))
        x = rng.standard_normal((2, cols))
        Y = sp.spmm_f64(h, torch_cuda.from_numpy(x).cuda()).cpu().numpy()
        for b in range(2):
            want = np.zeros(rows)
            for r in range(rows):
                acc = 0.0
                for e in range(ptr[r], ptr[r + 1]):
                    acc = acc + val[e] * x[b, idx[e]]
                want[r] = acc
            assert np.array_equal(u64(Y[b]), u64(want)), (layout, b)
    for layout in (0, 1):
        r = sp.read_sparse(want_text, layout)
        assert r.layout == layout and r.spec is None
        csr = r if layout == 0 else sp.relayout(r, 0)  # (CSC text is in column-major order)
        assert csr.write_text(transform_header=False) == want_text


def _csc(rows, cols, ptr, idx, val):
    trip = sorted((int(idx[e]), r, float(val[e])) for r in range(rows) for e in range(ptr[r], ptr[r + 1]))
    cptr = np.zeros(cols + 1, np.int64)
    for c, _, _ in trip:
        cptr[c + 1] += 1
    return np.cumsum(cptr), np.array([r for _, r, _ in trip], np.int64), np.array([v for _, _, v in trip])
