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
