"""GPU: the device verification sweep (inc/verify.hpp:59-169)
and the device comparators of inc/reference.hpp (direct_conv, im2col_conv).

The fp64 comparators must reproduce the reference's own functions BIT FOR BIT
(compared with the compiled reference / the restated direct_conv); the fp32
comparators must equal the device SpMV bit for bit; the sweep's counters must
equal the reference's run_verification on the same grid (golden.json)."""
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


SPECS = [(64, 64, 3, 1, 1), (257, 193, 5, 3, 4), (31, 40, 7, 2, 3), (12, 9, 11, 1, 5), (9, 9, 1, 2, 0)]


@pytest.mark.parametrize("spec", SPECS)
def test_direct_and_im2col_f64_bitexact_vs_reference(sp, orc, torch_cuda, spec):
    torch = torch_cuda
    m, n, k = spec[:3]
    kern, X = problem(orc, 41, m, n, k, batch=3)
    k64 = kern.astype(np.float64)
    A = torch.from_numpy(X.astype(np.float64)).cuda()
    T = torch.from_numpy(k64).cuda()
    cs = sp.ConvSpec(*spec)
    d = sp.direct_conv(cs, A, T).cpu().numpy()
    i = sp.im2col_conv(cs, A, T).cpu().numpy()
    for b in range(3):
        want = orc.direct_conv(*spec, X[b].astype(np.float64), k64)
        assert np.array_equal(d[b].view(np.uint64), want.view(np.uint64)), (spec, b)
        assert np.array_equal(i[b].view(np.uint64), want.view(np.uint64)), (spec, b)


def test_direct_f64_vs_compiled_reference(sp, ref, torch_cuda):
    torch = torch_cuda
    rng = np.random.default_rng(2)
    for spec in [(20, 17, 3, 1, 1), (33, 8, 4, 3, 2)]:
        m, n, k = spec[:3]
        a = rng.standard_normal(m * n)
        w = rng.standard_normal(k * k)
        got = sp.direct_conv(sp.ConvSpec(*spec), torch.from_numpy(a).cuda(), torch.from_numpy(w).cuda())
        want = ref.direct_conv(*spec, a, w)
        assert np.array_equal(got.cpu().numpy()[0].view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("spec", SPECS)
def test_f32_comparators_equal_spmv(sp, orc, torch_cuda, spec):
    """fp32 direct / im2col (fmaf, (j,i) order) == the SpMV of T, bit for bit."""
    torch = torch_cuda
    m, n, k = spec[:3]
    kern, X = problem(orc, 42, m, n, k, batch=4)
    t = sp.build_transform(sp.Kernel(k, kern.astype(np.float64)), sp.ConvSpec(*spec))
    Xd = torch.from_numpy(X).cuda()
    Y = sp.spmm(t, Xd)
    T = torch.from_numpy(kern).cuda()
    d = sp.direct_conv(sp.ConvSpec(*spec), Xd, T)
    i = sp.im2col_conv(sp.ConvSpec(*spec), Xd, T)
    torch.cuda.synchronize()
    y = Y.cpu().numpy().view(np.uint32)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), y)
    assert np.array_equal(i.cpu().numpy().view(np.uint32), y)


def test_verification_sweep_small_matches_reference(sp, golden):
    js, _ = golden
    want = js["run_verification_6x1"]
    rep = sp.run_verification(6, 1)
    assert rep["failures"] == 0, rep["failure_lines"]
    for key in ("specs", "conv_cases", "clipped_specs", "max_conv_dev", "max_layout_dev"):
        assert rep[key] == want[key], key  # the fp64 leg reproduces the reference's report
    assert rep["max_rel_dev"] <= 1e-5


@pytest.mark.slow
def test_verification_sweep_default_grid(sp, golden):
    """The reference's default sweep (max_dim 12, 3 seeds: 12,984 specs,
    38,952 convolution cases) on the device path."""
    js, _ = golden
    want = js["run_verification_12x3"]
    rep = sp.run_verification(12, 3)
    assert rep["failures"] == 0, rep["failure_lines"]
    for key in ("specs", "conv_cases", "clipped_specs", "max_conv_dev", "max_layout_dev"):
        assert rep[key] == want[key], key
    assert rep["max_rel_dev"] <= 1e-5


def test_reference_host_comparators_bitexact(sp, ref):
    """spconv_reference_host (host-buffer fp64 direct_conv / im2col_conv /
    im2col lowering, the drop-in reference.hpp's backend) == the compiled
    reference, bit for bit."""
    rng = np.random.default_rng(8)
    for spec in [(20, 17, 3, 1, 1), (33, 8, 4, 3, 2), (9, 9, 11, 1, 5)]:
        m, n, k, s, p = spec
        mo, no = (m + 2 * p - k) // s + 1, (n + 2 * p - k) // s + 1
        a = rng.standard_normal(m * n)
        w = rng.standard_normal(k * k)
        want = ref.direct_conv(*spec, a, w)
        for mode in (0, 1):
            out = np.empty(mo * no)
            sp._check(sp.lib.spconv_reference_host(mode, m, n, k, s, p, w.ctypes.data, a.ctypes.data,
                                                   out.ctypes.data, 0))
            assert np.array_equal(out.view(np.uint64), want.view(np.uint64)), (spec, mode)
        patches = np.empty(k * k * mo * no)
        sp._check(sp.lib.spconv_reference_host(2, m, n, k, s, p, None, a.ctypes.data, patches.ctypes.data, 0))
        pad = np.zeros((m + 2 * p, n + 2 * p))
        pad[p:p + m, p:p + n] = a.reshape(m, n)
        for j in range(k):
            for i in range(k):
                row = pad[j:j + s * (mo - 1) + 1:s, i:i + s * (no - 1) + 1:s].reshape(-1)
                assert np.array_equal(patches[(j * k + i) * mo * no:(j * k + i + 1) * mo * no], row)
