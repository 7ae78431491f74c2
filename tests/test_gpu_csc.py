"""GPU parity of the CSC layout: build_transform(...,
Layout::CSC) (inc/conv.hpp:179-204 with compile's CSC order, inc/sparse.hpp:
85-119), relayout (:268-274), CSC SpMV (:194-205), and the CSC text form.

Storage is compared BIT-EXACTLY with the reference's own CSC (golden digests
from the compiled reference) and with the oracle's restated transposition;
outputs bit-exactly with the fp32 ordered-fmaf restatement (the reference's
one-thread CSC scatter sums every output in the same column-ascending order
as the CSR loop -- its fp64 CSC and CSR outputs are identical, see
golden.json ``y_csc``)."""
import hashlib

import numpy as np
import pytest

from helpers import CONFIGS, CSC_BAND_KERNELS, golden_cases, problem, sha, sweep_specs, BAND_KERNELS

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


def build(sp, spec, kern, layout):
    return sp.build_transform(sp.Kernel(spec[2], np.asarray(kern, np.float64)), sp.ConvSpec(*spec),
                              layout=layout)


def bits(a):
    a = np.ascontiguousarray(a, np.float32)
    v = a.view(np.uint32).copy()
    v[np.isnan(a)] = 0x7FC00000
    return v


def csc_of(orc, spec, kern):
    """The oracle's CSC: restated transposition of the restated CSR build."""
    m, n = spec[:2]
    ptr, idx, val = orc.build_transform(*spec, np.asarray(kern, np.float64))
    return orc.transpose(ptr.size - 1, m * n, ptr, idx, val)


def apply(torch, sp, t, X, path=None):
    Xd = torch.from_numpy(np.ascontiguousarray(X, np.float32)).cuda()
    with sp.options(path=path):
        Y = sp.spmm(t, Xd)
    torch.cuda.synchronize()
    return Y.cpu().numpy()


def test_csc_config1_arrays(sp, golden):
    _, npz = golden
    t = build(sp, CONFIGS[0], npz["c1_kernel"], sp.Layout.CSC)
    assert t.layout == sp.Layout.CSC and t.major_dim == 64 * 64
    ptr, idx, val = t.export()
    assert np.array_equal(ptr, npz["c1_csc_ptr"]) and np.array_equal(idx, npz["c1_csc_idx"])
    assert np.array_equal(val.view(np.uint64), npz["c1_csc_val"].view(np.uint64))


def test_csc_build_matches_reference_digests(sp, orc, golden):
    """Config 2 + all 36 edge specs, normal and zero-tap kernels: the device
    CSC, widened, hashes to the reference's build_transform(.., CSC)."""
    js, _ = golden
    for key, spec, kern, _img in golden_cases(orc, js):
        t = build(sp, spec, kern, sp.Layout.CSC)
        assert sha(*t.export()) == js["digests"][key]["csc"], key


def test_csc_build_sweep_vs_oracle(sp, orc):
    """Every geometry of the m,n <= 9 grid (k up to 15), dense and zero-tap kernels."""
    rng = np.random.default_rng(12)
    for ci, spec in enumerate(sweep_specs(9)):
        if ci % 3:
            continue
        k = spec[2]
        kern = orc.random_normal_f32(orc.derive_seed(42, 3000 + ci), k * k).astype(np.float64)
        if ci % 2 == 0:
            kern[rng.random(k * k) < 0.35] = 0.0
        t = build(sp, spec, kern, sp.Layout.CSC)
        want = csc_of(orc, spec, kern)
        got = t.export()
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), spec
        assert np.array_equal(got[2].view(np.uint64), want[2].view(np.uint64)), spec


def test_csc_build_edge_values(sp, orc):
    """NaN / inf / -0 taps, p > k (padding-only rows), empty columns (s > k)."""
    cases = [((6, 7, 3, 1, 1), np.array([1, np.nan, 0, -0.0, 2, np.inf, 3, 0, -1])),
             ((5, 4, 2, 3, 4), np.arange(1, 5, dtype=np.float64)),
             ((20, 17, 2, 3, 0), np.array([1.0, -2.0, 3.0, 0.5])),
             ((9, 9, 3, 2, 2), np.zeros(9))]
    for spec, kern in cases:
        t = build(sp, spec, kern, sp.Layout.CSC)
        want = csc_of(orc, spec, kern)
        got = t.export()
        assert t.nnz == want[2].size, spec
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), spec
        assert np.array_equal(bits(got[2]), bits(want[2])), spec


@pytest.mark.slow
def test_csc_build_config3_full_size(sp, orc):
    spec = CONFIGS[2]
    kern = orc.random_normal_f32(orc.derive_seed(orc.derive_seed(42, 2), 1), 9)
    t = build(sp, spec, kern, sp.Layout.CSC)
    want = csc_of(orc, spec, kern)
    got = t.export()
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    assert np.array_equal(got[2].view(np.uint64), want[2].view(np.uint64))


@pytest.mark.parametrize("spec", [(64, 64, 3, 1, 1), (300, 260, 7, 2, 3), (257, 193, 5, 3, 4),
                                  (130, 68, 3, 2, 0)])
def test_csc_apply_bitexact(sp, orc, torch_cuda, spec):
    """A CSC transform applies bit-identically to the CSR ordered-fmaf chain,
    single vector (latency kernel) and batch (band / tiled path)."""
    m, n, k = spec[:3]
    kern, X = problem(orc, 31, m, n, k, batch=5)
    t = build(sp, spec, kern, sp.Layout.CSC)
    want = orc.spmm_native(*orc.build_native(*spec, kern), X)
    assert np.array_equal(bits(apply(torch_cuda, sp, t, X)), bits(want))
    assert np.array_equal(bits(apply(torch_cuda, sp, t, X[:1])), bits(want[:1]))
    assert np.array_equal(bits(apply(torch_cuda, sp, t, X, "generic")), bits(want))
    # and the fp64 reference semantics of convolve() on the CSC handle
    cp, ci, cv = csc_of(orc, spec, kern)
    y64 = orc.spmv_csc_f64(t.rows, cp, ci, cv, X[0].astype(np.float64))
    cond = orc.spmv_abs(*orc.build_transform(*spec, kern.astype(np.float64)), X[0].astype(np.float64))
    out = sp.convolve(t, X[0].astype(np.float64).reshape(m, n)).reshape(-1)
    assert np.all(np.abs(out - y64) <= 1e-5 * cond)


def test_relayout_roundtrip(sp, orc, torch_cuda):
    """relayout CSR -> CSC -> CSR on conv handles (device rebuild) and on
    generic uploads (host transposition): storage identical to the oracle's."""
    spec = (41, 37, 5, 2, 3)
    kern, X = problem(orc, 32, 41, 37, 5, batch=3)
    kern = kern.astype(np.float64)
    kern[3] = 0.0
    t = build(sp, spec, kern, sp.Layout.CSR)
    c = sp.relayout(t, sp.Layout.CSC)
    assert c.layout == sp.Layout.CSC and c.spec == t.spec
    want = csc_of(orc, spec, kern)
    assert all(np.array_equal(a, b) for a, b in zip(c.export(), want))
    back = sp.relayout(c, sp.Layout.CSR)
    assert all(np.array_equal(a, b) for a, b in zip(back.export(), t.export()))
    same = sp.relayout(t, sp.Layout.CSR)
    assert all(np.array_equal(a, b) for a, b in zip(same.export(), t.export()))
    # generic (host-uploaded) matrices
    ptr, idx, val = t.export()
    g = sp.Transform.from_host(t.rows, t.cols, ptr, idx, val)
    gc = sp.relayout(g, sp.Layout.CSC)
    assert gc.layout == sp.Layout.CSC
    assert all(np.array_equal(a, b) for a, b in zip(gc.export(), want))
    u = sp.Transform.from_host(t.rows, t.cols, *want, layout=sp.Layout.CSC)
    assert all(np.array_equal(a, b) for a, b in zip(u.export(), want))
    assert all(np.array_equal(a, b) for a, b in zip(sp.relayout(u, sp.Layout.CSR).export(), t.export()))
    wantY = orc.spmm_native(*orc.build_native(*spec, kern.astype(np.float32)), X)
    for h in (c, gc, u):
        assert np.array_equal(bits(apply(torch_cuda, sp, h, X)), bits(wantY))


def test_csc_upload_validation(sp):
    with pytest.raises(ValueError, match="strictly ascending per column"):
        sp.Transform.from_host(3, 2, np.array([0, 2, 3]), np.array([1, 0, 2]), np.ones(3),
                               layout=sp.Layout.CSC)
    with pytest.raises(ValueError, match="layout must be"):
        sp.Transform.from_host(3, 2, np.array([0, 0, 0]), np.array([], np.int64), np.array([]), layout=2)


def test_csc_text_bytes_match_reference(sp, golden):
    """write_transform of CSC transforms (column-major entry order, "csc"
    header) is byte-identical to the reference's."""
    js, _ = golden
    for case in js["text"]:
        m, n, k, s, p = case["spec"]
        kern = np.array(case["kernel_bits"], np.uint32).view(np.float32).astype(np.float64)
        t = build(sp, (m, n, k, s, p), kern, sp.Layout.CSC)
        data = t.write_text()
        assert len(data) == case["csc_bytes"], case["spec"]
        assert hashlib.sha256(data).hexdigest() == case["csc_sha"], (case["spec"], case["variant"])


def test_csc_text_read_back(sp, orc, ref, torch_cuda):
    """read_transform of a csc file (the reference's own bytes, and ours):
    layout CSC, storage identical, conv geometry adopted (band path)."""
    spec = (70, 52, 3, 1, 1)
    kern, X = problem(orc, 33, 70, 52, 3, batch=4)
    data = ref.build(*spec, kern.astype(np.float64), layout=1).write_text()
    r = sp.read_transform(data)
    assert r.layout == sp.Layout.CSC and r.spec == sp.ConvSpec(*spec)
    want = csc_of(orc, spec, kern)
    assert all(np.array_equal(a, b) for a, b in zip(r.export(), want))
    assert r.write_text() == data
    Y = apply(torch_cuda, sp, r, X)
    assert r.last_kernel in BAND_KERNELS + CSC_BAND_KERNELS
    assert np.array_equal(bits(Y), bits(orc.spmm_native(*orc.build_native(*spec, kern), X)))
    # a non-conv csc matrix stays generic but keeps its layout
    lines = data.split(b"\n")
    lines[7] = b" ".join(lines[7].split(b" ")[:2] + [b"0.5"])
    g = sp.read_transform(b"\n".join(lines))
    assert g.layout == sp.Layout.CSC
    gp, gi, gv = g.export()
    assert np.array_equal(gp, want[0]) and gv[4] == 0.5
