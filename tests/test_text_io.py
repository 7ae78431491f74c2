"""Transform persistence: write_transform / write_sparse
rendered on the GPU must be byte-identical to the reference's text
(inc/conv.hpp:217-244, inc/sparse.hpp:396-432, format_value inc/grid.hpp:54-59),
and read_transform must rebuild the same matrix with the reference's checks
and messages."""
import hashlib

import numpy as np
import pytest

from helpers import problem, zero_tap_kernel, BAND_KERNELS


def _sp():
    import paper_2411_19419_b200 as sp
    return sp


# ---------------------------------------------------------------------------
# CPU: every parse / validation error is raised before any device work.
# ---------------------------------------------------------------------------

BAD = [
    (b"", RuntimeError, r"^read_transform: bad header line$"),
    (b"%%transform 4 4 3 1 x csr\n", RuntimeError, r"^read_transform: bad header line$"),
    (b"%%transfrm 4 4 3 1 0 csr\n", RuntimeError, r"^read_transform: bad header line$"),
    (b"%%transform 4 4 9 1 0 csr\n", ValueError, r"^ConvSpec: kernel larger than padded input"),
    (b"%%transform 4 4 3 1 0 coo\n", ValueError, r"^unknown layout 'coo' \(expected csr or csc\)$"),
    (b"%%transform 4 4 3 1 0 csr\n%%sparse matrix\n", RuntimeError,
     r"^read_sparse: bad header line '%%sparse matrix'$"),
    (b"%%transform 4 4 3 1 0 csr\n%%sparse coordinate real\n4 16\n", RuntimeError,
     r"^read_sparse: bad 'rows cols nnz' line$"),
    (b"%%transform 4 4 3 1 0 csr\n%%sparse coordinate real\n4 16 2\n1 1 0.5\n", RuntimeError,
     r"^read_sparse: expected 2 entries, got 1$"),
    (b"%%transform 4 4 3 1 0 csr\n%%sparse coordinate real\n4 16 1\n5 1 0.5\n", ValueError,
     r"^Triplets: entry \(4, 0\) outside 4x16$"),
    (b"%%transform 4 4 3 1 0 csr\n%%sparse coordinate real\n4 16 2\n1 2 1\n1 2 3\n", ValueError,
     r"^SparseMatrix: duplicate entry at \(0, 1\)$"),
    (b"%%transform 4 4 3 1 0 csr\n%%sparse coordinate real\n5 16 0\n", RuntimeError,
     r"^read_transform: matrix is 5x16 but spec \(m=4, n=4, k=3, s=1, p=0\) requires 4x16$"),
    (b"%%transform 4 4 3 1 0 csr\n%%sparse coordinate real\n4 16 1\n1 1 nan\n", RuntimeError,
     r"^read_sparse: expected 1 entries, got 0$"),
]


@pytest.mark.parametrize("text,exc,msg", BAD)
def test_read_errors_match_reference(text, exc, msg):
    sp = _sp()
    with pytest.raises(exc, match=msg):
        sp.read_transform(text)


def test_read_errors_agree_with_compiled_reference(ref):
    """The same inputs through the reference's own read_transform."""
    from oracle import RefError
    for text, exc, msg in BAD:
        with pytest.raises(RefError, match=msg):
            ref.read_transform(text)


# ---------------------------------------------------------------------------
# GPU: byte parity of the device-rendered text
# ---------------------------------------------------------------------------

@pytest.mark.gpu
def test_write_transform_bytes_match_reference(orc, golden):
    sp = _sp()
    js, _ = golden
    for case in js["text"]:
        m, n, k, s, p = case["spec"]
        kern = np.array(case["kernel_bits"], np.uint32).view(np.float32)
        t = sp.build_transform(sp.Kernel(k, kern.astype(np.float64)), sp.ConvSpec(m, n, k, s, p))
        data = t.write_text()
        assert len(data) == case["bytes"], case["spec"]
        assert hashlib.sha256(data).hexdigest() == case["sha"], (case["spec"], case["variant"])


@pytest.mark.gpu
def test_format_g17_every_class_of_float(golden):
    """Exact %.17g of fp32 values widened to double (normals, subnormals,
    powers of ten, the 1e-4 / 1e17 style switches, +-0, +-inf, +-nan)."""
    sp = _sp()
    js, _ = golden
    bits = np.array([b for b, _ in js["g17"]], np.uint32)
    want = [w for _, w in js["g17"]]
    N = bits.size
    vals = bits.view(np.float32).astype(np.float64)
    t = sp.Transform.from_host(1, N, np.array([0, N]), np.arange(N), vals)
    lines = t.write_text(transform_header=False).decode().split("\n")
    assert lines[0] == "%%sparse coordinate real" and lines[1] == f"1 {N} {N}"
    got = [ln.split(" ")[2] for ln in lines[2:2 + N]]
    bad = [(hex(int(b)), g, w) for b, g, w in zip(bits, got, want) if g != w]
    assert not bad, bad[:10]


@pytest.mark.gpu
def test_read_transform_roundtrip_and_adoption(orc):
    """read(write(T)) rebuilds T exactly and comes back as a conv handle
    (the band kernels apply); a non-conv matrix stays generic."""
    sp = _sp()
    import torch
    spec = (130, 96, 5, 2, 2)
    kern, X = problem(orc, 21, 130, 96, 5, batch=6)
    t = sp.build_transform(sp.Kernel(5, kern.astype(np.float64)), sp.ConvSpec(*spec))
    data = t.write_text()
    r = sp.read_transform(data)
    assert r.spec == sp.ConvSpec(*spec)
    for a, b in zip(t.export(), r.export()):
        assert np.array_equal(a, b)
    assert r.write_text() == data
    Y = sp.spmm(r, torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    assert r.last_kernel in BAND_KERNELS
    want = orc.spmm_native(*orc.build_native(*spec, kern), X)
    assert np.array_equal(Y.cpu().numpy().view(np.uint32), want.view(np.uint32))
    # scramble one value: still read exactly, but generic
    lines = data.split(b"\n")
    lines[10] = b" ".join(lines[10].split(b" ")[:2] + [b"0.125"])
    g = sp.read_transform(b"\n".join(lines))
    ptr, idx, val = g.export()
    assert np.array_equal(ptr, t.export()[0]) and val[7] == 0.125
    sp.spmm(g, torch.from_numpy(X).cuda())
    assert g.last_kernel not in BAND_KERNELS


@pytest.mark.gpu
def test_read_reference_written_file(ref, orc):
    """A file the reference wrote (zero-tap kernel, unsorted entries allowed)
    reads back to the reference's own matrix."""
    sp = _sp()
    spec = (40, 33, 3, 1, 1)
    kern = zero_tap_kernel(orc, 3, 5).astype(np.float32).astype(np.float64)
    rt = ref.build(*spec, kern)
    data = rt.write_text()
    r = sp.read_transform(data)
    ptr, idx, val = rt.export()
    gp, gi, gv = r.export()
    assert np.array_equal(gp, ptr) and np.array_equal(gi, idx) and np.array_equal(gv, val)
    # entries in reverse order: compile() sorts them (inc/sparse.hpp:91-97)
    head, body = data.split(b"\n", 3)[:3], data.split(b"\n", 3)[3]
    rev = b"\n".join(head) + b"\n" + b"\n".join(reversed(body.strip().split(b"\n"))) + b"\n"
    r2 = sp.read_transform(rev)
    assert np.array_equal(r2.export()[1], idx)


def _glibc_g17(v):
    import ctypes
    libc = ctypes.CDLL(None)
    buf = ctypes.create_string_buffer(64)
    libc.snprintf(buf, 64, b"%.17g", ctypes.c_double(v))
    return buf.value.decode()


def test_format_g17_f64_matches_glibc():
    """The fp64 renderer (values a handle keeps exactly, spconv_format_g17 --
    the same code the device text writer runs) == glibc's %.17g, the
    reference's format_value (inc/grid.hpp:54-59): random bit patterns over
    the whole range, subnormals, the extremes, powers of ten and their
    neighbours, exact decimal ties, the fixed/exponent switches."""
    sp = _sp()
    rng = np.random.default_rng(1)
    vals = list(rng.integers(0, 2**64, 20000, dtype=np.uint64).view(np.float64))
    vals += list(rng.standard_normal(5000)) + list(rng.standard_normal(2000) * 1e-300)
    vals += list(rng.integers(1, 2**52, 2000, dtype=np.uint64).view(np.float64))  # subnormals
    for e in range(-325, 309):
        p = float(f"1e{e}")
        vals += [p, np.nextafter(p, 0), np.nextafter(p, np.inf)]
    vals += [5e-324, 2.2250738585072014e-308, 2.225073858507201e-308, 1.7976931348623157e308,
             0.0, -0.0, 1e-4, 9.9999999999999995e-5, 1e17, 99999999999999984.0, 1e16, 0.5, 2.5,
             0.1, 1 / 3, 2.0**-1074, 2.0**-1022, 2.0**1023, 123456789012345678.0, 9007199254740993.0]
    vals += [float(x) for x in range(1, 3000, 7)] + [x / 64 for x in range(-500, 500, 3)]
    bad = []
    for v in vals:
        v = float(v)
        if v != v or v in (float("inf"), float("-inf")):
            continue
        g, w = sp.format_g17(v), _glibc_g17(v)
        if g != w:
            bad.append((v.hex(), g, w))
    assert not bad, bad[:10]
    for v, w in [(float("inf"), "inf"), (float("-inf"), "-inf"), (float("nan"), "nan"), (-float("nan"), "-nan")]:
        assert sp.format_g17(v) == w == _glibc_g17(v)
