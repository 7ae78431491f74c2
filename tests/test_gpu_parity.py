"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Structure (row_ptr, col_idx) and values of T are compared BIT-EXACTLY with the
restatement and, through the golden digests, with the compiled reference's own
output.  SpMV/SpMM outputs are compared bit-exactly with the fp32 ordered-fmaf
restatement of spmv_csr_rows (inc/sparse.hpp:180-192) -- the device kernels
accumulate each row in the same column-ascending order -- and, against the
fp64 reference, within the north-star tolerance:
    |y_gpu - y_ref| <= 1e-5 * sum_e |val_e * x_col_e|   (condition-aware relative).
"""
import os

import numpy as np
import pytest

from helpers import LATENCY_SPEC, CONFIGS, golden_cases, problem, sha, sweep_specs, zero_tap_kernel, BAND_KERNELS

pytestmark = pytest.mark.gpu

TOL = 1e-5  # relative fp32 tolerance of BASELINE.json north_star


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture(scope="module")
def sp(torch_cuda):
    import paper_2411_19419_b200 as sp
    return sp


def native_copy(t):
    ptr = np.empty(t.rows + 1, np.int32)
    idx = np.empty(max(t.nnz, 1), np.int32)
    val = np.empty(max(t.nnz, 1), np.float32)
    t.copy_native(ptr, idx, val)
    return ptr, idx[: t.nnz], val[: t.nnz]


def build(sp, spec, kern):
    return sp.build_transform(sp.Kernel(spec[2], np.asarray(kern, np.float64)), sp.ConvSpec(*spec))


def bits(a):
    """fp32 bit patterns, with every NaN canonicalised (the GPU's default NaN is
    0x7fffffff, x86's 0x7fc00000/0xffc00000; payloads are not part of the contract)."""
    a = np.ascontiguousarray(a, np.float32)
    v = a.view(np.uint32).copy()
    v[np.isnan(a)] = 0x7FC00000
    return v


def assert_same_csr(t, ref_csr):
    ptr, idx, val = native_copy(t)
    rp, ri, rv = ref_csr
    assert np.array_equal(ptr, rp.astype(np.int32))
    assert np.array_equal(idx, ri.astype(np.int32))
    assert np.array_equal(bits(val), bits(rv.astype(np.float32)))


def run_spmm(torch, sp, t, X, path=None, ldx_pad=0):
    """X host f32 [B, cols] -> device SpMM -> host [B, rows]."""
    B, cols = X.shape
    Xd = torch.zeros(B, cols + ldx_pad, dtype=torch.float32, device="cuda")
    Xd[:, :cols] = torch.from_numpy(X)
    with sp.options(path=path):
        Y = sp.spmm(t, Xd[:, :cols])
    torch.cuda.synchronize()
    return Y.cpu().numpy()


# ---------------------------------------------------------------------------
# CSR build
# ---------------------------------------------------------------------------

def test_build_config1_matches_reference_arrays(sp, golden):
    _, npz = golden
    t = build(sp, CONFIGS[0], npz["c1_kernel"])
    ptr, idx, val = t.export()
    assert np.array_equal(ptr, npz["c1_ptr"]) and np.array_equal(idx, npz["c1_idx"])
    assert np.array_equal(val.view(np.uint64), npz["c1_val"].view(np.uint64))


def test_build_zero_tap_fixture(sp, golden):
    _, npz = golden
    t = build(sp, (3, 3, 3, 1, 1), npz["zt_kernel"])
    ptr, idx, val = t.export()
    assert np.array_equal(ptr, npz["zt_ptr"]) and np.array_equal(idx, npz["zt_idx"])
    assert np.array_equal(val, npz["zt_val"])


def test_build_matches_reference_digests(sp, orc, golden):
    """Config 2 and every config-5 edge spec (normal + zero-tap kernels): the
    device CSR, widened, hashes to the reference's own digest."""
    js, _ = golden
    for key, spec, kern, _img in golden_cases(orc, js):
        t = build(sp, spec, kern)
        d = js["digests"][key]
        assert t.nnz == d["nnz"], key
        assert sha(*t.export()) == d["csr"], key


def test_build_sweep_vs_oracle(sp, orc):
    """Every geometry of the m,n <= 9 verify grid, with all-non-zero and zero-tap kernels."""
    rng = np.random.default_rng(11)
    for ci, spec in enumerate(sweep_specs(9)):
        k = spec[2]
        kern = orc.random_normal_f32(orc.derive_seed(42, 1000 + ci), k * k)
        if ci % 4 == 0:
            kern[rng.random(k * k) < 0.35] = 0.0
        t = build(sp, spec, kern)
        assert_same_csr(t, orc.build_native(*spec, kern))


def test_build_edge_cases(sp, orc):
    # empty rows (k=1, p=1: the whole border is padding), p > k, all-zero kernel, NaN taps
    cases = [((257, 193, 1, 1, 1), np.ones(1, np.float32)),
             ((5, 4, 2, 3, 4), np.arange(1, 5, dtype=np.float32)),
             ((9, 9, 3, 2, 2), np.zeros(9, np.float32)),
             ((6, 7, 3, 1, 1), np.array([1, np.nan, 0, -0.0, 2, np.inf, 3, 0, -1], np.float32)),
             ((1, 1, 1, 1, 3), np.array([2.5], np.float32))]
    for spec, kern in cases:
        t = build(sp, spec, kern)
        rp, ri, rv = orc.build_native(*spec, kern)
        ptr, idx, val = native_copy(t)
        assert np.array_equal(ptr, rp) and np.array_equal(idx, ri)
        assert np.array_equal(bits(val), bits(rv))
        assert t.nnz == rv.size


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [2, 3])
def test_build_full_size(sp, orc, cfg):
    """Configs 3 (1024^2 k3) and 4 (4096^2 k7 s2 p3, 205 M entries) bit-exact."""
    spec = CONFIGS[cfg]
    kern = orc.random_normal_f32(orc.derive_seed(orc.derive_seed(42, cfg), 1), spec[2] ** 2)
    t = build(sp, spec, kern)
    assert t.nnz == orc.nnz_bound(*spec)
    ptr, idx, val = native_copy(t)
    rp, ri, rv = orc.build_native(*spec, kern)
    assert np.array_equal(ptr, rp)
    assert np.array_equal(idx, ri)
    assert np.array_equal(bits(val), bits(rv))
    # closed form: row counts are Theorem 2.1's per-output counts
    assert np.array_equal(np.diff(ptr.astype(np.int64)), orc.nnz_per_output(*spec))


# ---------------------------------------------------------------------------
# SpMV / SpMM
# ---------------------------------------------------------------------------

def test_spmv_config1_vs_reference_y(sp, orc, golden, torch_cuda):
    _, npz = golden
    t = build(sp, CONFIGS[0], npz["c1_kernel"])
    x = npz["c1_image"].astype(np.float32)
    y = sp.spmv(t, torch_cuda.from_numpy(x).cuda()).cpu().numpy()
    ptr, idx, val = npz["c1_ptr"], npz["c1_idx"], npz["c1_val"]
    assert np.array_equal(bits(y), bits(orc.spmv_f32_fma(ptr, idx, val, x)))
    cond = orc.spmv_abs(ptr, idx, val, npz["c1_image"])
    assert np.all(np.abs(y - npz["c1_y"]) <= TOL * cond)


def test_spmv_config2_all_paths(sp, orc, torch_cuda):
    m, n, k, s, p = CONFIGS[1]
    kern, X = problem(orc, 1, m, n, k, batch=1)
    t = build(sp, CONFIGS[1], kern)
    rp, ri, rv = orc.build_native(*CONFIGS[1], kern)
    want = orc.spmm_native(rp, ri, rv, X)
    for path in (None, "spmv", "spmv_plain", "banded", "tiled", "tiled_notma", "generic"):
        Y = run_spmm(torch_cuda, sp, t, X, path)
        assert np.array_equal(bits(Y), bits(want)), path
    # fp64 reference tolerance
    y64 = orc.spmv_f64(rp.astype(np.int64), ri.astype(np.int64), rv.astype(np.float64), X[0].astype(np.float64))
    cond = orc.spmv_abs(rp.astype(np.int64), ri.astype(np.int64), rv.astype(np.float64), X[0].astype(np.float64))
    assert np.all(np.abs(want[0] - y64) <= TOL * cond)


@pytest.mark.parametrize("batch", [1, 2, 3, 5, 8, 13, 32])
def test_spmm_batches_and_tails(sp, orc, torch_cuda, batch):
    spec = (96, 72, 5, 2, 2)
    kern, X = problem(orc, 7, 96, 72, 5, batch=batch)
    t = build(sp, spec, kern)
    want = orc.spmm_native(*orc.build_native(*spec, kern), X)
    for path in (None, "spmv", "spmv_plain", "banded", "tiled", "tiled_notma", "generic"):
        assert np.array_equal(bits(run_spmm(torch_cuda, sp, t, X, path)), bits(want)), path
    # padded leading dimension (ldx = cols + 4 keeps TMA-legal 16B strides)
    assert np.array_equal(bits(run_spmm(torch_cuda, sp, t, X, None, ldx_pad=4)), bits(want))


def test_spmm_golden_specs(sp, orc, golden, torch_cuda):
    """Every digest case (config 2 + 36 edge specs x {normal, zero-tap}): SpMM of
    3 images bit-exact vs the ordered-fmaf oracle; image 0 within tolerance of
    the reference fp64 output (its digest pins the oracle's fp64 y)."""
    js, _ = golden
    for key, spec, kern, img in golden_cases(orc, js):
        m, n = spec[0], spec[1]
        _, Xo = problem(orc, 9, m, n, 1, batch=2)
        X = np.concatenate([img[None].astype(np.float32), Xo])
        t = build(sp, spec, kern)
        rp, ri, rv = orc.build_native(*spec, kern.astype(np.float32))
        want = orc.spmm_native(rp, ri, rv, X)
        Y = run_spmm(torch_cuda, sp, t, X)
        assert np.array_equal(bits(Y), bits(want)), key
        ptr, idx, val = orc.build_transform(*spec, kern)
        y64 = orc.spmv_f64(ptr, idx, val, img)
        assert sha(y64) == js["digests"][key]["y"], key
        cond = orc.spmv_abs(ptr, idx, val, img)
        assert np.all(np.abs(Y[0] - y64) <= TOL * cond + 1e-37), key


def test_spmm_sweep_small(sp, orc, torch_cuda):
    for ci, spec in enumerate(sweep_specs(7)):
        if ci % 3:
            continue
        m, n, k = spec[:3]
        kern = orc.random_normal_f32(orc.derive_seed(42, 5000 + ci), k * k)
        X = np.stack([orc.random_normal_f32(orc.derive_seed(42, 9000 + ci + b), m * n) for b in range(3)])
        t = build(sp, spec, kern)
        want = orc.spmm_native(*orc.build_native(*spec, kern), X)
        assert np.array_equal(bits(run_spmm(torch_cuda, sp, t, X)), bits(want)), spec


BANDED = [(3, 1), (5, 1), (3, 2), (5, 2), (7, 2)]


@pytest.mark.parametrize("ks", BANDED)
def test_banded_borders_and_fallback(sp, orc, torch_cuda, ks):
    """Register-blocked kernel on border-heavy shapes (partial tiles, p > 0, odd
    sizes with n % 4 == 0), and its in-kernel fallback: a zero tap or a NaN tap
    makes every tile fail the band check and take the per-entry loop."""
    k, s = ks
    rng = np.random.default_rng(k * 10 + s)
    for (m, n, p) in [(33, 36, k // 2), (70, 44, 0), (19, 20, k - 1), (k, 8, 1)]:
        spec = (m, n, k, s, p)
        if orc.spec_check(*spec):
            continue
        kern = orc.random_normal_f32(orc.derive_seed(77, m * n + k), k * k)
        X = rng.standard_normal((9, m * n)).astype(np.float32)
        X[3, rng.integers(0, m * n)] = np.inf
        for variant in ("dense", "zero", "nan"):
            kv = kern.copy()
            if variant == "zero":
                kv[k * k // 2] = 0.0
            elif variant == "nan":
                kv[0] = np.nan
            t = build(sp, spec, kv)
            want = orc.spmm_native(*orc.build_native(*spec, kv), X)
            for path in (None, "banded"):
                Y = run_spmm(torch_cuda, sp, t, X, path)
                assert np.array_equal(bits(Y), bits(want)), (spec, variant, path)


def test_spmm_nonfinite_inputs(sp, orc, torch_cuda):
    """inf/NaN pixels only reach the outputs whose rows store them (no 0*inf leaks)."""
    spec = (32, 32, 3, 1, 1)
    kern, X = problem(orc, 3, 32, 32, 3, batch=4)
    X[0, 5] = np.inf
    X[1, 100] = np.nan
    X[2, 1023] = -np.inf
    t = build(sp, spec, kern)
    want = orc.spmm_native(*orc.build_native(*spec, kern), X)
    for path in (None, "spmv", "spmv_plain", "banded", "tiled", "tiled_notma", "generic"):
        Y = run_spmm(torch_cuda, sp, t, X, path)
        assert np.array_equal(bits(Y), bits(want)), path


@pytest.mark.slow
def test_spmm_config3_full_size(sp, orc, torch_cuda):
    m, n, k, s, p = CONFIGS[2]
    kern, X = problem(orc, 2, m, n, k, batch=12)
    t = build(sp, CONFIGS[2], kern)
    want = orc.spmm_native(*orc.build_native(*CONFIGS[2], kern), X)
    assert np.array_equal(bits(run_spmm(torch_cuda, sp, t, X)), bits(want))


@pytest.mark.slow
def test_spmm_config4_full_size(sp, orc, torch_cuda):
    m, n, k, s, p = CONFIGS[3]
    kern, X = problem(orc, 3, m, n, k, batch=3)
    t = build(sp, CONFIGS[3], kern)
    rp, ri, rv = orc.build_native(*CONFIGS[3], kern)
    want = orc.spmm_native(rp, ri, rv, X)
    Y = run_spmm(torch_cuda, sp, t, X)
    assert np.array_equal(bits(Y), bits(want))


def test_generic_csr_upload(sp, orc, torch_cuda):
    """Arbitrary host CSR (not a conv transform) through the generic kernel."""
    rng = np.random.default_rng(3)
    rows, cols = 300, 517
    ptr = [0]
    idx, val = [], []
    for r in range(rows):
        c = np.sort(rng.choice(cols, size=int(rng.integers(0, 40)), replace=False))
        idx += c.tolist()
        val += rng.standard_normal(c.size).astype(np.float32).tolist()
        ptr.append(len(idx))
    ptr, idx, val = np.array(ptr, np.int64), np.array(idx, np.int64), np.array(val, np.float64)
    t = sp.Transform.from_host(rows, cols, ptr, idx, val)
    X = rng.standard_normal((4, cols)).astype(np.float32)
    want = orc.spmm_f32_fma(ptr, idx, val, X)
    assert np.array_equal(bits(run_spmm(torch_cuda, sp, t, X)), bits(want))
    assert np.array_equal(t.export()[1], idx)
    for b in (1, 2):  # latency kernel (warp per 32 rows) on ragged rows, empty rows included
        for path in (None, "spmv_plain"):
            assert np.array_equal(bits(run_spmm(torch_cuda, sp, t, X[:b], path)), bits(want[:b])), (b, path)
        assert t.last_kernel == "csr_spmv_unrolled"
        assert np.array_equal(bits(run_spmm(torch_cuda, sp, t, X[:b])), bits(want[:b]))
        assert t.last_kernel == "csr_spmv_bulk"


@pytest.mark.parametrize("kernel", ["rowblock", "plain"])
def test_generic_multivector_kernels(sp, orc, torch_cuda, kernel, opts):
    """Batches on a generic CSR: the row-block kernel (matrix staged once per
    CTA, images four at a time) and the thread-per-row kernel
    (option generic=plain), ragged and empty rows, row blocks that end
    mid-matrix, batches that are not a multiple of four, padded ldx,
    non-finite inputs; rows longer than 64 entries take the plain kernel."""
    if kernel == "plain":
        opts(generic="plain")
    rng = np.random.default_rng(5)
    for rows, cols, maxlen in ((300, 517, 40), (1000, 2000, 64), (77, 5000, 100)):
        lens = rng.integers(0, maxlen + 1, rows)
        lens[::7] = 0
        ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        idx = np.concatenate([np.sort(rng.choice(cols, size=int(L), replace=False)) for L in lens]).astype(np.int64)
        val = rng.standard_normal(idx.size)
        val[::11] = 0.0
        t = sp.Transform.from_host(rows, cols, ptr, idx, val)
        for batch in (3, 6, 13):
            X = rng.standard_normal((batch, cols)).astype(np.float32)
            X[1, rng.integers(0, cols)] = np.inf
            want = orc.spmm_f32_fma(ptr, idx, val, X)
            for pad in (0, 4):
                got = run_spmm(torch_cuda, sp, t, X, ldx_pad=pad)
                assert np.array_equal(bits(got), bits(want)), (rows, batch, pad)
            expect = "csr_spmm_rowblock" if kernel == "rowblock" and maxlen <= 64 else "csr_spmm_generic"
            assert t.last_kernel == expect


def test_end_to_end_host_path(sp, orc, torch_cuda):
    """convolve_batch on host buffers (chunked H2D / SpMM / D2H pipeline)."""
    spec = (256, 200, 3, 1, 1)
    kern, X = problem(orc, 8, 256, 200, 3, batch=70)
    t = build(sp, spec, kern)
    want = orc.spmm_native(*orc.build_native(*spec, kern), X)
    Y = sp.convolve_batch(t, X)
    assert np.array_equal(bits(Y), bits(want))
    Xp = torch_cuda.from_numpy(X).pin_memory()
    Yp = sp.convolve_batch(t, Xp)
    assert np.array_equal(bits(Yp.numpy()), bits(want))


@pytest.mark.parametrize("spec", [(56, 56, 3, 1, 1), (224, 224, 7, 2, 3), (14, 14, 1, 1, 0), (28, 28, 2, 2, 0),
                                  (7, 7, 3, 1, 1), (30, 30, 5, 3, 2)])
def test_host_path_single_images(sp, orc, torch_cuda, spec):
    """Single images (and pairs) on host buffers -- the DenseNet call shape.
    Page-locked Y: the kernel writes y straight into host memory; pageable
    buffers: copies both ways.  Bit-exact either way."""
    m, n, k = spec[:3]
    kern, X = problem(orc, 9, m, n, k, batch=2)
    t = build(sp, spec, kern)
    want = orc.spmm_native(*orc.build_native(*spec, kern), X)
    for b in (1, 2):
        Xp = torch_cuda.from_numpy(X[:b].copy()).pin_memory()
        Yp = torch_cuda.empty(b, t.rows).pin_memory()
        sp.convolve_batch(t, Xp, Yp)
        assert np.array_equal(bits(Yp.numpy()), bits(want[:b])), (spec, b, t.last_kernel)
        Y = sp.convolve_batch(t, X[:b].copy())  # pageable
        assert np.array_equal(bits(Y), bits(want[:b])), (spec, b)


@pytest.mark.slow
def test_config3_auto_path_bench_batches(sp, orc, torch_cuda):
    """BASELINE config 3 through the default (auto) path at the bench's
    per-GPU batches -- 96 and 32 images, the fused check-and-apply --
    images {0, b/2, b-1} bit-exact vs the oracle."""
    spec = (1024, 1024, 3, 1, 1)
    kern, X = problem(orc, 2, 1024, 1024, 3, batch=3)
    t = build(sp, spec, kern)
    ptr, idx, val = orc.build_native(*spec, kern)
    for batch in (96, 32):
        Xd = torch_cuda.from_numpy(np.repeat(X, (batch + 2) // 3, axis=0)[:batch]).cuda()
        Y = sp.spmm(t, Xd)
        torch_cuda.cuda.synchronize()
        assert t.last_kernel in BAND_KERNELS, t.last_kernel
        for i in (0, batch // 2, batch - 1):
            want = orc.spmm_native(ptr, idx, val, Xd[i].cpu().numpy()[None])[0]
            assert np.array_equal(bits(Y[i].cpu().numpy()), bits(want)), (batch, i)


def test_reference_semantics_convolve(sp, orc, golden):
    """The fp64-in/fp64-out convolve() mirror computes in fp64 with the
    reference's rounding: BIT-identical to the reference's convolve() on
    config 1 (fp32-representable taps)."""
    _, npz = golden
    t = build(sp, CONFIGS[0], npz["c1_kernel"])
    out = sp.convolve(t, npz["c1_image"].reshape(64, 64))
    assert out.shape == (64, 64)
    assert np.array_equal(out.reshape(-1).view(np.uint64), npz["c1_y"].view(np.uint64))
    assert t.last_kernel == "csr_spmm_f64"
    with pytest.raises(ValueError, match=r"^convolve: input is 3x64 but transform expects \(m=64"):
        sp.convolve(t, np.zeros((3, 64)))


def test_errors(sp, torch_cuda):
    t = build(sp, (8, 8, 3, 1, 1), np.ones(9, np.float32))
    x = torch_cuda.zeros(63, device="cuda")
    with pytest.raises(ValueError, match="spmv: matrix has 64 columns but vector has 63 elements"):
        sp.spmv(t, x)
    with pytest.raises(ValueError, match="leading dimension"):
        sp._check(sp.lib.spconv_spmm(t._h, x.data_ptr(), 10, x.data_ptr(), 64, 1, None))
    with pytest.raises(ValueError, match="build_conv_matrix: kernel side 2 does not match"):
        sp.build_transform(sp.Kernel(2, np.ones(4)), sp.ConvSpec(8, 8, 3, 1, 1))
    buf = torch_cuda.zeros(3 * 64, device="cuda")  # in place / overlapping: rejected, nothing launched
    with pytest.raises(ValueError, match="spconv_spmv: x and y overlap"):
        sp._check(sp.lib.spconv_spmv(t._h, buf.data_ptr(), buf.data_ptr() + 4 * 10, None))
    with pytest.raises(ValueError, match="spconv_spmm: X and Y overlap"):
        sp._check(sp.lib.spconv_spmm(t._h, buf.data_ptr(), 64, buf.data_ptr() + 4 * 100, 64, 2, None))
    sp._check(sp.lib.spconv_spmm(t._h, buf.data_ptr(), 64, buf.data_ptr() + 4 * 128, 64, 1, None))  # disjoint


@pytest.mark.parametrize("spec", [(1024, 1024, 3, 1, 1), (512, 512, 5, 2, 2), (300, 260, 7, 2, 3),
                                  (200, 132, 5, 1, 2), (130, 68, 3, 2, 0)])
def test_band_path_is_default(sp, orc, torch_cuda, spec):
    """Dense taps on a band geometry: the auto path is the two-kernel band path
    (CSR band check + register-blocked apply), bit-exact vs the oracle, with
    unaligned output rows (n_out % 4 != 0) and padded ldy included."""
    m, n, k = spec[:3]
    kern, X = problem(orc, 11, m, n, k, batch=5)
    t = build(sp, spec, kern)
    want = orc.spmm_native(*orc.build_native(*spec, kern), X)
    Y = run_spmm(torch_cuda, sp, t, X)
    assert t.last_kernel in BAND_KERNELS
    assert np.array_equal(bits(Y), bits(want)), spec
    # ldy padded by one float: Y rows lose 16-byte alignment -> scalar stores
    Xd = torch_cuda.from_numpy(X).cuda()
    Yd = torch_cuda.full((5, t.rows + 1), -7.0, device="cuda")
    sp.spmm(t, Xd, Yd[:, : t.rows])
    torch_cuda.cuda.synchronize()
    Yh = Yd.cpu().numpy()
    assert np.array_equal(bits(Yh[:, : t.rows]), bits(want))
    assert np.all(Yh[:, t.rows] == -7.0)  # nothing written past the row


@pytest.mark.parametrize("fused", ["0", "1"])
def test_band_concurrent_streams(sp, orc, torch_cuda, fused, opts):
    """One immutable handle applied on two streams at once (the band check's
    per-segment bytes are rewritten with identical values: benign), with the
    check kernel and with the fused check-and-apply."""
    opts(fused=fused)
    spec = (256, 256, 3, 1, 1)
    kern, X = problem(orc, 12, 256, 256, 3, batch=16)
    t = build(sp, spec, kern)
    want = orc.spmm_native(*orc.build_native(*spec, kern), X)
    Xd = torch_cuda.from_numpy(X).cuda()
    s1, s2 = torch_cuda.cuda.Stream(), torch_cuda.cuda.Stream()
    torch_cuda.cuda.synchronize()
    outs = []
    for _ in range(20):
        Y1 = torch_cuda.empty(16, t.rows, device="cuda")
        Y2 = torch_cuda.empty(16, t.rows, device="cuda")
        sp.spmm(t, Xd, Y1, stream=s1)
        sp.spmm(t, Xd, Y2, stream=s2)
        outs += [Y1, Y2]
    torch_cuda.cuda.synchronize()
    for Y in outs:
        assert np.array_equal(bits(Y.cpu().numpy()), bits(want))


@pytest.mark.parametrize("stage", ["window", "bulk"])
@pytest.mark.parametrize("skew", [1, -1, 3])
def test_spmv_spec_mispredicted_rows(sp, orc, torch_cuda, skew, stage):
    """The latency SpMV's closed-form run prediction never decides the result:
    with the predicted run bounds deliberately skewed (test hook), every warp
    takes the reload path and the output is still bit-exact (the windowed
    kernel and the bulk-staged one)."""
    spec = (64, 48, 5, 2, 2)
    kern, X = problem(orc, 13, 64, 48, 5, batch=2)
    t = build(sp, spec, kern)
    want = orc.spmm_native(*orc.build_native(*spec, kern), X)
    with sp.options(spec_skew=skew, stage=stage):
        Y = run_spmm(torch_cuda, sp, t, X)
    assert t.last_kernel == ("conv_spmv_win" if stage == "window" else "csr_spmv_bulk<spec>")
    assert np.array_equal(bits(Y), bits(want))


class _DevArray:
    """A raw device pointer seen as a 1-D CUDA array (test access to a handle's arrays)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3}


@pytest.mark.parametrize("check", ["same", "fused"])
@pytest.mark.parametrize("spec", [(256, 256, 3, 1, 1), (300, 260, 7, 2, 3)])
def test_band_check_reads_the_matrix(sp, orc, torch_cuda, spec, check, opts):
    """The band path re-reads T on every call: entries altered in device memory
    after the build (a value, a column moved far outside its tile's input
    window, a column moved to an earlier image row) are picked up by the next
    spmm -- the affected segments fail the check and take the per-entry loop --
    and the output is bit-exact vs the oracle on the altered CSR."""
    # check kernel on the caller's stream / fused into the apply
    opts(fused="1" if check == "fused" else "0")
    m, n, k = spec[:3]
    kern, X = problem(orc, 14, m, n, k, batch=6)
    t = build(sp, spec, kern)
    ptr, idx, val = native_copy(t)
    clean = run_spmm(torch_cuda, sp, t, X)
    assert np.array_equal(bits(clean), bits(orc.spmm_native(ptr, idx, val, X)))
    assert t.band_check_status()[1] == 0  # the untouched matrix passes every segment
    _, ci, cv = t.device_ptrs()
    dci = torch_cuda.as_tensor(_DevArray(ci, t.nnz, "<i4"), device="cuda")
    dcv = torch_cuda.as_tensor(_DevArray(cv, t.nnz, "<f4"), device="cuda")
    no = sp.ConvSpec(*spec).n_out
    r1 = (t.rows // 2) + no // 2           # interior rows
    r2 = (t.rows // 3) + 5
    r3 = (2 * t.rows // 3) + no // 3
    e_last = int(ptr[r1 + 1]) - 1          # last entry of r1 -> 40 image rows further down
    e_first = int(ptr[r2])                 # first entry of r2 -> 40 image rows up
    e_val = int(ptr[r3]) + 2
    idx[e_last] += 40 * n
    idx[e_first] -= 40 * n
    val[e_val] = np.float32(val[e_val] * 3.0)
    assert 0 <= idx[e_first] and idx[e_last] < m * n
    dci[e_last] = int(idx[e_last])
    dci[e_first] = int(idx[e_first])
    dcv[e_val] = float(val[e_val])
    torch_cuda.cuda.synchronize()
    Y = run_spmm(torch_cuda, sp, t, X)
    assert t.last_kernel in BAND_KERNELS
    assert 1 <= t.band_check_status()[1] <= 3  # only the tampered segments failed
    want = orc.spmm_native(ptr, idx, val, X)
    assert not np.array_equal(bits(want), bits(clean))
    assert np.array_equal(bits(Y), bits(want))


@pytest.mark.parametrize("batch", [1, 6])
def test_stream_ordered_change_of_handed_out_storage(sp, orc, torch_cuda, batch):
    """A value changed by a kernel of the caller's on the same stream, with no
    synchronisation before the next apply: stream order alone must make the
    apply see it.  (Applies read the matrix before griddepcontrol.wait only
    when launched as programmatic dependents, which storage handed out by
    device_ptrs never is.)"""
    torch = torch_cuda
    spec = (256, 256, 3, 1, 1)
    kern, X = problem(orc, 15, 256, 256, 3, batch=batch)
    t = build(sp, spec, kern)
    ptr, idx, val = native_copy(t)
    Xd = torch.from_numpy(X).cuda()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):  # (the handle is past its first apply: PDL would be allowed)
            sp.spmm(t, Xd, stream=st)
        _, _, cv = t.device_ptrs()
        dcv = torch.as_tensor(_DevArray(cv, t.nnz, "<f4"), device="cuda")
        for rep in range(4):
            e = int(ptr[t.rows // 2 + 17 * rep]) + 1
            val[e] = np.float32(val[e] * -3.0 + 0.5)
            torch.cuda._sleep(200_000)  # (the caller's kernel runs long enough to overlap a PDL launch)
            dcv[e] = float(val[e])      # a kernel on st
            Y = sp.spmm(t, Xd, stream=st)
            st.synchronize()
            want = orc.spmm_native(ptr, idx, val, X)
            assert np.array_equal(bits(Y.cpu().numpy()), bits(want)), (batch, rep, t.last_kernel)


@pytest.mark.parametrize("bulk_store", ["0", "1"])
@pytest.mark.parametrize("variant", ["block", "warp", "persist"])
def test_build_variants_bitexact(sp, orc, variant, bulk_store, opts):
    """The CSR build kernels (block scan / warp-local / persistent, option build), with
    the staged entries written back by TMA bulk stores or by 16-byte stores
    (option bulk_store), give the oracle's arrays for every unrolled k,
    dense and zero-tap kernels; so does the CSC build."""
    rng = np.random.default_rng(21)
    opts(bulk_store=bulk_store, build=variant)
    if True:
        for spec in [(70, 45, 1, 1, 1), (130, 97, 3, 1, 1), (64, 80, 5, 2, 2), (101, 77, 7, 2, 3),
                     (48, 50, 11, 3, 10), (33, 20, 3, 2, 0)]:
            k = spec[2]
            for zero in (False, True):
                kern = rng.standard_normal(k * k).astype(np.float32)
                if zero:
                    kern[rng.random(k * k) < 0.3] = 0.0
                t = build(sp, spec, kern)
                assert_same_csr(t, orc.build_native(*spec, kern))
                tc = sp.build_transform(sp.Kernel(k, kern.astype(np.float64)), sp.ConvSpec(*spec),
                                        layout=sp.Layout.CSC)
                ptr, idx, val = orc.build_transform(*spec, kern.astype(np.float64))
                want = orc.transpose(ptr.size - 1, spec[0] * spec[1], ptr, idx, val)
                got = tc.export()
                assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
                assert np.array_equal(got[2].view(np.uint64), want[2].view(np.uint64))


@pytest.mark.parametrize("stage", ["bulk", "window", "auto"])
def test_latency_spmv_staging_variants(sp, orc, torch_cuda, stage, opts):
    """Both stagings of the latency SpMV (bulk copies / per-lane 16-byte
    loads, option stage), dense-tap (closed-form run) and zero-tap
    (row_ptr-driven) transforms, batch 1 and 2: bit-exact."""
    rng = np.random.default_rng(31)
    opts(stage=stage)
    if True:
        for spec in [(512, 512, 5, 2, 2), (97, 130, 3, 1, 1), (64, 72, 7, 2, 3), (33, 35, 5, 3, 4)]:
            m, n, k = spec[:3]
            kern, X = problem(orc, 51, m, n, k, batch=2)
            for zero in (False, True):
                kv = kern.copy()
                if zero:
                    kv[rng.random(k * k) < 0.3] = 0.0
                t = build(sp, spec, kv)
                want = orc.spmm_native(*orc.build_native(*spec, kv), X)
                for b in (1, 2):
                    Y = run_spmm(torch_cuda, sp, t, X[:b])
                    assert t.last_kernel in LATENCY_SPEC
                    assert np.array_equal(bits(Y), bits(want[:b])), (spec, zero, b)


@pytest.mark.parametrize("batch", [1, 2, 6])
def test_spmm_misaligned_buffers(sp, orc, torch_cuda, batch):
    """X and Y one float off 16-byte alignment (TMA can't describe X; Y can't
    take vector stores): every path still bit-exact, nothing written outside Y."""
    torch = torch_cuda
    spec = (64, 64, 3, 1, 1)
    kern, X = problem(orc, 16, 64, 64, 3, batch=batch)
    t = build(sp, spec, kern)
    want = orc.spmm_native(*orc.build_native(*spec, kern), X)
    xb = torch.zeros(batch * t.cols + 1, device="cuda")
    xb[1:] = torch.from_numpy(X.reshape(-1)).cuda()
    yb = torch.full((batch * t.rows + 2,), -3.0, device="cuda")
    Xd = xb[1:].view(batch, t.cols)
    Yd = yb[1:-1].view(batch, t.rows)
    for path in (None, "tiled", "generic"):
        with sp.options(path=path):
            sp.spmm(t, Xd, Yd)
        torch.cuda.synchronize()
        got = yb.cpu().numpy()
        assert got[0] == -3.0 and got[-1] == -3.0, path
        assert np.array_equal(bits(got[1:-1].reshape(batch, t.rows)), bits(want)), path


@pytest.mark.parametrize("spec,batch", [((256, 256, 3, 1, 1), 6), ((300, 260, 7, 2, 3), 3), ((512, 512, 5, 2, 2), 1)])
def test_spmm_in_cuda_graph(sp, orc, torch_cuda, spec, batch):
    """spmm captured into a CUDA graph (the band check then stays on the
    captured stream) and replayed on new inputs: bit-exact."""
    torch = torch_cuda
    m, n, k = spec[:3]
    kern, X = problem(orc, 17, m, n, k, batch=2 * batch)
    t = build(sp, spec, kern)
    want = orc.spmm_native(*orc.build_native(*spec, kern), X)
    Xd = torch.from_numpy(X[:batch]).cuda()
    Yd = torch.empty(batch, t.rows, device="cuda")
    cs = torch.cuda.Stream()
    sp.spmm(t, Xd, Yd, stream=cs)  # warm (attributes, workspaces) outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        sp.spmm(t, Xd, Yd, stream=cs)
    Xd.copy_(torch.from_numpy(X[batch:]))
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(bits(Yd.cpu().numpy()), bits(want[batch:]))


@pytest.mark.parametrize("fused", ["0", "1"])
@pytest.mark.parametrize("spec", [(1024, 1024, 3, 1, 1), (200, 132, 5, 1, 2), (130, 68, 3, 2, 0),
                                  (300, 260, 7, 2, 3), (97, 64, 5, 2, 2), (64, 40, 3, 1, 1)])
def test_band_fused_and_two_kernel(sp, orc, torch_cuda, spec, fused, opts):
    """The fused check-and-apply (segments checked by the producer warps, a
    fixup pass after) and the two-kernel form give the same bit-exact results
    on every band geometry, including grids with more CTAs than work items."""
    opts(fused=fused)
    m, n, k = spec[:3]
    kern, X = problem(orc, 18, m, n, k, batch=5)
    t = build(sp, spec, kern)
    Y = run_spmm(torch_cuda, sp, t, X)
    assert t.last_kernel == BAND_KERNELS[int(fused)]
    assert np.array_equal(bits(Y), bits(orc.spmm_native(*orc.build_native(*spec, kern), X)))


def test_fp64_path_bitexact_vs_reference_digests(sp, orc, golden, torch_cuda):
    """The fp64 device SpMV (reference arithmetic) reproduces the reference's
    own fp64 convolve() output BIT FOR BIT for config 2 and all 36 config-5
    edge specs, normal and zero-tap kernels (golden SHA-256 digests), and
    the CSC handle gives the same bits."""
    js, _ = golden
    for key, spec, kern, img in golden_cases(orc, js):
        m, n = spec[:2]
        t = build(sp, spec, kern)
        y = sp.convolve(t, img.reshape(m, n)).reshape(-1)
        assert sha(y) == js["digests"][key]["y"], key
        X = torch_cuda.from_numpy(np.stack([img, img[::-1].copy()])).cuda()
        Y = sp.spmm_f64(t, X).cpu().numpy()
        assert sha(Y[0]) == js["digests"][key]["y"], key
        ptr, idx, val = orc.build_transform(*spec, kern)
        assert np.array_equal(Y[1].view(np.uint64), orc.spmv_f64(ptr, idx, val, img[::-1].copy()).view(np.uint64))
    tc = sp.build_transform(sp.Kernel(5, kern if spec[2] == 5 else np.ones(25)), sp.ConvSpec(40, 36, 5, 2, 2),
                            layout=sp.Layout.CSC)
    tr = sp.relayout(tc, sp.Layout.CSR)
    a = np.linspace(-1, 1, 40 * 36).reshape(40, 36)
    assert np.array_equal(sp.convolve(tc, a).view(np.uint64), sp.convolve(tr, a).view(np.uint64))


def test_band_apply_captured_in_a_graph(sp, orc, torch_cuda):
    """Back-to-back band applies (programmatic dependent launches after the
    first) captured in a CUDA graph and replayed: every replay's outputs are the
    oracle's, with the inputs rewritten between replays."""
    torch = torch_cuda
    spec = (256, 256, 3, 1, 1)
    kern, X = problem(orc, 16, 256, 256, 3, batch=8)
    t = build(sp, spec, kern)
    ptr, idx, val = native_copy(t)
    Xd = torch.from_numpy(X).cuda()
    Ys = [torch.empty(8, t.rows, device="cuda") for _ in range(3)]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        sp.spmm(t, Xd, Ys[0], stream=st)  # (first apply outside the graph)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for Y in Ys:
            sp.spmm(t, Xd, Y, stream=st)
    for rep in range(3):
        Xn = X * (1.0 + rep) - rep
        Xd.copy_(torch.from_numpy(Xn.astype(np.float32)))
        g.replay()
        torch.cuda.synchronize()
        want = orc.spmm_native(ptr, idx, val, Xn.astype(np.float32))
        for Y in Ys:
            assert np.array_equal(bits(Y.cpu().numpy()), bits(want)), rep


@pytest.mark.parametrize("fused", ["0", "1"])
def test_programmatic_launch_modes_agree(sp, orc, torch_cuda, fused, opts):
    """Back-to-back band applies with the programmatic dependent launch on
    (both kernels / the apply only) and off give the oracle's bits every time,
    the output buffer rewritten by each call."""
    torch = torch_cuda
    spec = (384, 256, 3, 1, 1)
    kern, X = problem(orc, 17, 384, 256, 3, batch=12)
    t = build(sp, spec, kern)
    ptr, idx, val = native_copy(t)
    want = orc.spmm_native(ptr, idx, val, X)
    Xd = torch.from_numpy(X).cuda()
    Y = torch.empty(12, t.rows, device="cuda")
    for pdl in ("auto", "apply_only", "off", "auto"):
        opts(pdl=pdl, fused=fused)
        for _ in range(4):
            Y.fill_(float("nan"))
            sp.spmm(t, Xd, Y)
        torch.cuda.synchronize()
        assert np.array_equal(bits(Y.cpu().numpy()), bits(want)), (pdl, fused)
