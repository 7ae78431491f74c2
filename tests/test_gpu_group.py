"""GPU: the grouped apply (spconv_spmv_group / spconv_convolve_host_group,
csrc/group.cu) -- a list of transforms, each with its own vector, in one
launch -- gives every member bit for bit what spconv_spmv gives it, and the
oracle's ordered-fmaf row loop (the reference's spmv_csr_rows,
inc/sparse.hpp:180-192, in fp32)."""
import numpy as np
import pytest

from helpers import problem

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


# DenseNet121-like members plus odd shapes, strides and zero taps
SPECS = [(7, 7, 3, 1, 1), (56, 56, 3, 1, 1), (224, 224, 7, 2, 3), (14, 14, 1, 1, 0), (28, 28, 2, 2, 0),
         (33, 17, 5, 2, 2), (9, 130, 3, 3, 1), (112, 112, 3, 1, 1), (1, 1, 1, 1, 0), (64, 64, 11, 1, 5)]


def members(sp, orc, extra_csc=True):
    ts, xs, want = [], [], []
    for i, spec in enumerate(SPECS):
        m, n, k, s, p = spec
        kern, X = problem(orc, 60 + i, m, n, k)
        if i % 3 == 2:
            kern = kern.copy()
            kern[0] = 0.0  # a zero tap: fewer entries per row
        t = sp.build_transform(sp.Kernel(k, kern.astype(np.float64)), sp.ConvSpec(*spec))
        ts.append(t)
        xs.append(X[0])
        want.append(orc.spmm_native(*orc.build_native(*spec, kern.astype(np.float32)), X[:1])[0])
    # a matrix that is not a conv transform (host CSR upload)
    rng = np.random.default_rng(7)
    rows, cols = 300, 500
    cnt = rng.integers(0, 20, rows)
    ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    idx = np.concatenate([np.sort(rng.choice(cols, c, replace=False)) for c in cnt]).astype(np.int64)
    val = rng.standard_normal(ptr[-1])
    ts.append(sp.Transform.from_host(rows, cols, ptr, idx, val))
    x = rng.standard_normal(cols).astype(np.float32)
    xs.append(x)
    want.append(orc.spmm_native(ptr.astype(np.int32), idx.astype(np.int32), val.astype(np.float32), x[None])[0])
    if extra_csc:  # CSC storage: applied by its own kernel inside the call
        spec = (40, 40, 3, 1, 1)
        kern, X = problem(orc, 80, 40, 40, 3)
        ts.append(sp.build_transform(sp.Kernel(3, kern.astype(np.float64)), sp.ConvSpec(*spec), layout=1))
        xs.append(X[0])
        want.append(orc.spmm_native(*orc.build_native(*spec, kern), X[:1])[0])
    return ts, xs, want


def test_group_matches_spmv_and_oracle(sp, orc, torch_cuda):
    torch = torch_cuda
    ts, xs, want = members(sp, orc)
    xd = [torch.from_numpy(x).cuda() for x in xs]
    ys = sp.spmv_group(ts, xd)
    torch.cuda.synchronize()
    for i, (t, y, w) in enumerate(zip(ts, ys, want)):
        assert np.array_equal(bits(y.cpu().numpy()), bits(w)), i
        if t.layout == sp.Layout.CSR:
            assert t.last_kernel == "csr_spmv_group"
        one = sp.spmv(t, xd[i])
        torch.cuda.synchronize()
        assert np.array_equal(bits(one.cpu().numpy()), bits(w)), i


def test_group_host(sp, orc, torch_cuda):
    ts, xs, want = members(sp, orc)
    for _ in range(2):  # (second call: the staging is reused)
        ys = sp.convolve_group(ts, xs)
        for i, (y, w) in enumerate(zip(ys, want)):
            assert np.array_equal(bits(y), bits(w)), i


def test_group_nonfinite_and_many(sp, orc, torch_cuda):
    """More members than one launch holds (300 > 128), non-finite inputs."""
    torch = torch_cuda
    ts, xs, want = [], [], []
    rng = np.random.default_rng(3)
    for i in range(300):
        m = int(rng.integers(1, 20))
        k = int(rng.choice([1, 3, 5]))
        spec = (m, m, k, 1, k // 2)
        kern = rng.standard_normal(k * k).astype(np.float32)
        x = rng.standard_normal(m * m).astype(np.float32)
        if i % 50 == 7:
            x[0] = np.inf
        if i % 50 == 9:
            x[-1] = np.nan
        ts.append(sp.build_transform(sp.Kernel(k, kern.astype(np.float64)), sp.ConvSpec(*spec)))
        xs.append(x)
        want.append(orc.spmm_native(*orc.build_native(*spec, kern), x[None])[0])
    ys = sp.spmv_group(ts, [torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    for i, (y, w) in enumerate(zip(ys, want)):
        assert np.array_equal(bits(y.cpu().numpy()), bits(w)), i
    yh = sp.convolve_group(ts, xs)
    for i, (y, w) in enumerate(zip(yh, want)):
        assert np.array_equal(bits(y), bits(w)), i


def test_group_follows_altered_storage(sp, orc, torch_cuda):
    """The grouped kernel reads the stored entries: a value changed through
    device_ptrs shows up in the output."""
    torch = torch_cuda
    spec = (16, 16, 3, 1, 1)
    kern, X = problem(orc, 90, 16, 16, 3)
    t = sp.build_transform(sp.Kernel(3, kern.astype(np.float64)), sp.ConvSpec(*spec))
    rp, ci, va = t.export()
    _, _, vptr = t.device_ptrs()
    torch.cuda.synchronize()
    dv = torch.as_tensor(_DevArray(vptr, t.nnz, "<f4"), device="cuda")
    dv[5] = 2.5
    torch.cuda.synchronize()
    va = va.astype(np.float32)
    va[5] = 2.5
    want = orc.spmm_native(rp.astype(np.int32), ci.astype(np.int32), va, X[:1])[0]
    y = sp.spmv_group([t], [torch.from_numpy(X[0]).cuda()])[0]
    torch.cuda.synchronize()
    assert np.array_equal(bits(y.cpu().numpy()), bits(want))


def test_group_argument_errors(sp, orc, torch_cuda):
    torch = torch_cuda
    ts, xs, _ = members(sp, orc, extra_csc=False)
    xd = [torch.from_numpy(x).cuda() for x in xs]
    with pytest.raises(ValueError):
        sp.spmv_group(ts[:2], xd[:1])
    # y of member 0 overlapping member 1's x
    y0 = xd[1][: ts[0].rows] if ts[0].rows <= xd[1].numel() else None
    if y0 is not None:
        ys = [y0, torch.empty(ts[1].rows, device="cuda")]
        with pytest.raises(ValueError, match="overlaps"):
            sp.spmv_group(ts[:2], xd[:2], ys)
    assert sp.spmv_group([], []) == []


def u64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def test_group_f64_bitexact_vs_reference(sp, ref, torch_cuda):
    """fp64 grouped apply (device and host forms): every member bit-identical to
    the compiled reference's convolve() -- double taps incl. a zero and a
    1e-300 tap (exact values kept), CSR and CSC members in one call."""
    torch = torch_cuda
    specs = [(7, 7, 3, 1, 1), (56, 56, 3, 1, 1), (224, 224, 7, 2, 3), (14, 14, 1, 1, 0), (33, 17, 5, 2, 2),
             (64, 64, 11, 1, 5), (40, 40, 3, 1, 1)]
    ts, xs, want = [], [], []
    for i, spec in enumerate(specs):
        m, n, k = spec[:3]
        kern = ref.random_normal_kernel(k, 20 + i)
        if k > 1:
            kern[1] = 0.0
            kern[0] = 1e-300
        x = ref.random_normal_grid(m, n, 200 + i).reshape(-1)
        ts.append(sp.build_transform(sp.Kernel(k, kern), sp.ConvSpec(*spec), layout=1 if i == len(specs) - 1 else 0))
        xs.append(x)
        want.append(ref.build(*spec, kern).convolve(x[None])[0])
    ys = sp.spmv_group(ts, [torch.from_numpy(x).cuda() for x in xs])
    torch.cuda.synchronize()
    for i, (y, w) in enumerate(zip(ys, want)):
        assert np.array_equal(u64(y.cpu().numpy()), u64(w)), i
    assert ts[0].last_kernel == "csr_spmv_group<f64>"
    for _ in range(2):
        yh = sp.convolve_group_f64(ts, xs)
        for i, (y, w) in enumerate(zip(yh, want)):
            assert np.array_equal(u64(y), u64(w)), i


def test_group_empty_matrix_member(sp, orc, torch_cuda):
    """An all-zero kernel (no stored entries: every output +0.0) among other
    members, fp32 and fp64, device and host forms."""
    torch = torch_cuda
    specs = [(12, 12, 3, 1, 1), (20, 20, 5, 2, 2), (9, 9, 3, 1, 1)]
    kerns = [np.zeros(9), np.random.default_rng(1).standard_normal(25), np.random.default_rng(2).standard_normal(9)]
    ts = [sp.build_transform(sp.Kernel(sp_[2], kk), sp.ConvSpec(*sp_)) for sp_, kk in zip(specs, kerns)]
    assert ts[0].nnz == 0
    xs = [np.random.default_rng(10 + i).standard_normal(t.cols).astype(np.float32) for i, t in enumerate(ts)]
    ys = sp.spmv_group(ts, [torch.from_numpy(x).cuda() for x in xs])
    yh = sp.convolve_group(ts, xs)
    y64 = sp.convolve_group_f64(ts, [x.astype(np.float64) for x in xs])
    torch.cuda.synchronize()
    assert np.array_equal(bits(ys[0].cpu().numpy()), np.zeros(ts[0].rows, np.uint32))
    assert np.array_equal(bits(yh[0]), np.zeros(ts[0].rows, np.uint32))
    assert np.array_equal(u64(y64[0]), np.zeros(ts[0].rows, np.uint64))
    for i in (1, 2):
        one = sp.spmv(ts[i], torch.from_numpy(xs[i]).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(bits(ys[i].cpu().numpy()), bits(one.cpu().numpy()))
        assert np.array_equal(bits(yh[i]), bits(one.cpu().numpy()))
