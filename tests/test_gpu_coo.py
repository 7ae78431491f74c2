"""SparseMatrix::compile(Triplets, layout) on the device (spconv_matrix_from_coo,
inc/sparse.hpp:35-119): any insertion order -> the reference's compressed
storage (sorted by (major, minor), explicit zeros kept), duplicates rejected
with the reference's message (the first duplicate in the layout's sorted
order), exact doubles kept; then applied by the generic kernels.  Checked
against the compiled reference where it is present (Ref.write_sparse_csr of
the same triplets), else against a numpy restatement."""
import numpy as np
import pytest

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


def compressed(rows, cols, r, c, v, csc):
    order = np.lexsort((r, c)) if csc else np.lexsort((c, r))
    major = (c if csc else r)[order]
    ptr = np.zeros((cols if csc else rows) + 1, np.int64)
    np.add.at(ptr, major + 1, 1)
    return np.cumsum(ptr), (r if csc else c)[order], v[order]


def u64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("shape", [(1, 1, 1), (37, 53, 300), (1000, 700, 20000), (5, 9000, 4000), (64, 64, 0)])
def test_compile_matches_restatement(sp, orc, torch_cuda, layout, shape):
    rows, cols, n = shape
    rng = np.random.default_rng(rows * 7 + n)
    flat = rng.choice(rows * cols, size=min(n, rows * cols), replace=False)
    r, c = (flat // cols).astype(np.int64), (flat % cols).astype(np.int64)
    v = rng.standard_normal(r.size)
    v[::5] = 0.0   # explicit zeros are kept
    v[1::7] = -0.0
    if r.size > 3:
        v[2] = 1e-310  # a double fp32 cannot hold
    t = sp.compile_triplets(rows, cols, r, c, v, layout)
    assert t.layout == layout and t.nnz == r.size
    gp, gi, gv = t.export()
    wp, wi, wv = compressed(rows, cols, r, c, v, layout == 1)
    assert np.array_equal(gp, wp) and np.array_equal(gi[:r.size], wi)
    assert np.array_equal(u64(gv[:r.size]), u64(wv))
    # applied through the generic kernels, row-major arrays from the same compile
    if r.size:
        x = rng.standard_normal((5, cols)).astype(np.float32)
        Y = sp.spmm(t, torch_cuda.from_numpy(x).cuda()).cpu().numpy()
        p, i, val = compressed(rows, cols, r, c, v, False)
        want = orc.spmm_f32_fma(p, i, val, x)
        assert np.array_equal(Y.view(np.uint32), want.view(np.uint32))


def test_compile_matches_reference(sp, ref):
    rng = np.random.default_rng(3)
    rows, cols = 40, 31
    flat = rng.choice(rows * cols, size=200, replace=False)
    r, c = (flat // cols).astype(np.int64), (flat % cols).astype(np.int64)
    v = rng.standard_normal(200)
    t = sp.compile_triplets(rows, cols, r, c, v)
    p, i, val = compressed(rows, cols, r, c, v, False)
    assert t.write_text(transform_header=False) == ref.write_sparse_csr(rows, cols, p, i, val)


@pytest.mark.parametrize("layout,want", [(0, "(2, 4)"), (1, "(3, 1)")])
def test_duplicates_rejected_like_compile(sp, layout, want):
    """Two duplicated coordinates: compile() names the first in ITS sorted
    order -- row-major for CSR, column-major for CSC."""
    import re
    r = np.array([3, 0, 2, 3, 2, 5])
    c = np.array([1, 0, 4, 1, 4, 2])
    with pytest.raises(ValueError, match="^" + re.escape("SparseMatrix: duplicate entry at " + want) + "$"):
        sp.compile_triplets(6, 6, r, c, np.ones(6), layout)


# ---------------------------------------------------------------------------
# spgemm and the factor matrices (inc/sparse.hpp:296-342, inc/conv.hpp:125-162)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("spec", [(9, 7, 3, 1, 1), (20, 17, 5, 2, 2), (12, 9, 4, 3, 2), (6, 6, 1, 1, 2)])
@pytest.mark.parametrize("double_taps", [False, True])
def test_spgemm_route_equals_build_transform(sp, ref, spec, double_taps):
    """The reference's Spgemm route: spgemm(build_conv_matrix, build_padding_matrix)
    == build_transform, bit for bit -- zero taps dropped by the accumulator,
    exact doubles kept -- and == the reference's own build."""
    m, n, k, s, p = spec
    rng = np.random.default_rng(k * 11 + s)
    kern = rng.standard_normal(k * k)
    if not double_taps:
        kern = kern.astype(np.float32).astype(np.float64)
    if k > 1:
        kern[0] = 0.0
        kern[-1] = -0.0
    cs = sp.ConvSpec(*spec)
    C = sp.build_conv_matrix(sp.Kernel(k, kern), cs)
    P = sp.build_padding_matrix(cs)
    assert (C.rows, C.cols, C.nnz) == (cs.m_out * cs.n_out, (m + 2 * p) * (n + 2 * p), cs.m_out * cs.n_out * k * k)
    assert (P.rows, P.cols, P.nnz) == ((m + 2 * p) * (n + 2 * p), m * n, m * n)
    T = sp.spgemm(C, P)
    B = sp.build_transform(sp.Kernel(k, kern), cs)
    for a, b in zip(T.export(), B.export()):
        assert np.array_equal(a.view(np.uint64) if a.dtype == np.float64 else a,
                              b.view(np.uint64) if b.dtype == np.float64 else b)
    rp, ri, rv = ref.build(*spec, kern).export()
    gp, gi, gv = T.export()
    assert np.array_equal(gp, rp) and np.array_equal(gi[:rp[-1]], ri) and np.array_equal(u64(gv[:rp[-1]]), u64(rv))
    Tc = sp.spgemm(C, P, layout=1)
    assert Tc.layout == 1 and np.array_equal(Tc.export()[0], ref.build(*spec, kern, layout=1).export()[0])


def test_spgemm_random_matches_gustavson(sp):
    """Random operands with cancellations and zeros: the reference's Gustavson
    loop restated in Python (sequential fp64 sums in A-then-B order)."""
    rng = np.random.default_rng(12)
    def rand(rows, cols, dens):
        d = rng.standard_normal((rows, cols)) * (rng.random((rows, cols)) < dens)
        d[rng.random((rows, cols)) < 0.05] = 0.0
        ptr = np.concatenate([[0], np.cumsum((d != 0).sum(1))]).astype(np.int64)
        idx = np.nonzero(d)[1].astype(np.int64)
        return ptr, idx, d[d != 0]
    ap, ai, av = rand(33, 40, 0.2)
    bp, bi, bv = rand(40, 27, 0.25)
    bv[::9] = -av[0] if av.size else 1.0  # invite exact cancellations
    A = sp.Transform.from_host(33, 40, ap, ai, av)
    B = sp.Transform.from_host(40, 27, bp, bi, bv)
    G = sp.spgemm(A, B)
    want_p, want_i, want_v = [0], [], []
    for i in range(33):
        acc, order = {}, []
        for ka in range(ap[i], ap[i + 1]):
            k, a = ai[ka], av[ka]
            for kb in range(bp[k], bp[k + 1]):
                j = bi[kb]
                if j not in acc:
                    acc[j] = 0.0
                    order.append(j)
                acc[j] = acc[j] + a * bv[kb]
        for j in sorted(order):
            if acc[j] != 0.0:
                want_i.append(j)
                want_v.append(acc[j])
        want_p.append(len(want_i))
    gp, gi, gv = G.export()
    assert np.array_equal(gp, want_p) and np.array_equal(gi[:len(want_i)], want_i)
    assert np.array_equal(u64(gv[:len(want_v)]), u64(np.array(want_v)))
    with pytest.raises(ValueError, match=r"^spgemm: inner dimensions differ, 40 vs 33$"):
        sp.spgemm(A, G)
