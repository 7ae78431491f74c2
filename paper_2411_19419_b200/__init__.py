"""B200-native conv-as-SpMV (arXiv 2411.19419) -- Python front-end over the C ABI.

The product is ``libspconv_b200.so`` (hand-written sm_100a CUDA kernels behind
the extern "C" boundary in ``include/spconv_b200.h``).  This module is a thin
ctypes mirror of the reference's C++ operator API (namespace ``spconv`` in
/root/reference/proj/include/spconv): ``ConvSpec``, ``Kernel``, ``Transform``,
``build_transform``, ``convolve``, ``spmv`` keep the reference names, argument
meaning and error behaviour (``ValueError`` where the reference throws
``std::invalid_argument``, ``RuntimeError`` for ``std::runtime_error``/CUDA).
Device tensors are torch CUDA tensors (plumbing only); every arithmetic
operation on them runs in the CUDA library.  There is no CPU fallback: if the
library is missing, importing this package raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "ConvSpec", "Kernel", "Transform", "build_transform", "convolve", "convolve_batch",
    "spmv", "spmm", "spmm_f64", "convolve_batch_f64", "nnz_bound", "read_transform", "relayout", "Layout", "layout_name",
    "layout_from_name", "derive_seed", "random_normal", "set_option", "get_option", "options", "direct_conv", "im2col_conv", "run_verification", "library_path", "lib",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "libspconv_b200.so")

if not os.path.exists(library_path):
    raise ImportError(
        f"{library_path} is missing: build it with `make` (or __graft_entry__.build()); "
        "there is no CPU fallback for the conv-as-SpMV path")

lib = C.CDLL(library_path)

_i64 = C.c_int64
_vp = C.c_void_p
_P = C.POINTER


def _decl(name, args, res=C.c_int):
    f = getattr(lib, name)
    f.argtypes = args
    f.restype = res
    return f


_decl("spconv_last_error", [], C.c_char_p)
_decl("spconv_abi_version", [])
_decl("spconv_spec_check", [_i64] * 5)
_decl("spconv_nnz_bound", [_i64] * 5 + [_P(_i64)])
_decl("spconv_build_csr", [_i64] * 5 + [_vp, C.c_int, _vp, _P(_vp)])
_decl("spconv_csr_from_host", [_i64, _i64, _vp, _vp, _vp, C.c_int, _vp, _P(_vp)])
_decl("spconv_csr_shape", [_vp, _P(_i64), _P(_i64), _P(_i64)])
_decl("spconv_csr_spec", [_vp, _vp])
_decl("spconv_csr_device_ptrs", [_vp, _P(_vp), _P(_vp), _P(_vp)])
_decl("spconv_csr_export", [_vp, _vp, _vp, _vp])
_decl("spconv_csr_copy", [_vp, _vp, _vp, _vp, _vp])
_decl("spconv_spmv", [_vp, _vp, _vp, _vp])
_decl("spconv_spmm", [_vp, _vp, _i64, _vp, _i64, _i64, _vp])
_decl("spconv_convolve_host", [_vp, _vp, _vp, _i64])
_decl("spconv_convolve_host_f64", [_vp, _vp, _vp, _i64])
_decl("spconv_spmm_f64", [_vp, _vp, _i64, _vp, _i64, _i64, _vp])
_decl("spconv_csr_storage_bytes", [_vp, _P(_i64)])
_decl("spconv_band_check_flags", [_vp, _vp, _i64, _P(_i64)])
_decl("spconv_spmv_group", [_vp, _i64, _vp, _vp, _vp])
_decl("spconv_convolve_host_group", [_vp, _i64, _vp, _vp])
_decl("spconv_spmv_group_f64", [_vp, _i64, _vp, _vp, _vp])
_decl("spconv_convolve_host_group_f64", [_vp, _i64, _vp, _vp])
_decl("spconv_spmm_f64_threads", [_vp, _vp, _i64, _vp, _i64, _i64, C.c_int, _vp])
_decl("spconv_convolve_host_f64_threads", [_vp, _vp, _vp, _i64, C.c_int])
_decl("spconv_csr_last_kernel", [_vp], C.c_char_p)
_decl("spconv_band_check_status", [_vp, _P(_i64), _P(_i64)])
_decl("spconv_csr_write_text", [_vp, C.c_int, _vp, _i64, _P(_i64)])
_decl("spconv_transform_read", [_vp, _i64, C.c_int, _vp, _P(_vp)])
_decl("spconv_sparse_read", [_vp, _i64, C.c_int, C.c_int, _vp, _P(_vp)])
_decl("spconv_matrix_from_coo", [_i64, _i64, _i64, _vp, _vp, _vp, C.c_int, C.c_int, _vp, _P(_vp)])
_decl("spconv_spgemm", [_vp, _vp, C.c_int, _vp, _P(_vp)])
_decl("spconv_build_padding_matrix", [_i64] * 5 + [C.c_int, C.c_int, _vp, _P(_vp)])
_decl("spconv_build_conv_matrix", [_i64] * 5 + [_vp, C.c_int, C.c_int, _vp, _P(_vp)])
_decl("spconv_csr_free", [_vp])
_decl("spconv_build_transform", [_i64] * 5 + [_vp, C.c_int, C.c_int, _vp, _P(_vp)])
_decl("spconv_build_transform_f64", [_i64] * 5 + [_vp, C.c_int, C.c_int, _vp, _P(_vp)])
_decl("spconv_format_g17", [C.c_double, C.c_char_p])
_decl("spconv_csr_layout", [_vp, _P(C.c_int)])
_decl("spconv_relayout", [_vp, C.c_int, _vp, _P(_vp)])
_decl("spconv_direct_conv", [_i64] * 5 + [C.c_int, _vp, _vp, _vp, _vp, _i64, _vp])
_decl("spconv_im2col_conv", [_i64] * 5 + [C.c_int, _vp, _vp, _vp, _vp, _i64, _vp])
_decl("spconv_derive_seed", [C.c_uint64, C.c_uint64], C.c_uint64)
_decl("spconv_random_normal", [C.c_uint64, _i64, _vp])
_decl("spconv_reference_host", [C.c_int] + [_i64] * 5 + [_vp, _vp, _vp, C.c_int])
_decl("spconv_run_verification", [_i64, C.c_int, C.c_uint64, C.c_int, _vp, _vp, _vp, _i64])
_decl("spconv_matrix_from_host", [_i64, _i64, C.c_int, _vp, _vp, _vp, C.c_int, _vp, _P(_vp)])
_decl("spconv_set_option", [C.c_char_p, C.c_char_p])
_decl("spconv_get_option", [C.c_char_p, C.c_char_p, _i64])


def derive_seed(base: int, index: int) -> int:
    """derive_seed (inc/rng.hpp): the reference's per-problem seed derivation."""
    return int(lib.spconv_derive_seed(base, index))


def random_normal(seed: int, count: int, out=None) -> np.ndarray:
    """`count` standard normals of the reference's generator seeded by `seed`
    (random_normal_grid / random_normal_kernel, inc/rng.hpp:80-92), float64.
    Host code in the library (releases the GIL: callable from worker threads)."""
    if out is None:
        out = np.empty(count, np.float64)
    assert out.dtype == np.float64 and out.flags.c_contiguous and out.size >= count
    _check(lib.spconv_random_normal(seed, count, out.ctypes.data))
    return out


def set_option(name: str, value) -> None:
    """Process-wide kernel-path option (spconv_set_option, include/spconv_b200.h):
    forces an alternative kernel for cross-checks and A/B timing."""
    _check(lib.spconv_set_option(name.encode(), str(value).encode()))


def get_option(name: str) -> str:
    buf = C.create_string_buffer(64)
    _check(lib.spconv_get_option(name.encode(), buf, 64))
    return buf.value.decode()


class options:
    """Context manager: ``with options(path="tiled", fused=1): ...`` sets the
    options for the block and restores the previous values after it."""

    def __init__(self, **kw):
        self.kw = {k: v for k, v in kw.items() if v is not None}
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            set_option(k, v)
        return False


class Layout:
    """Storage layout (inc/sparse.hpp:24): CSR = 0, CSC = 1."""
    CSR = 0
    CSC = 1


def layout_name(layout: int) -> str:
    """inc/sparse.hpp:26."""
    return "csr" if layout == Layout.CSR else "csc"


def layout_from_name(s: str) -> int:
    """inc/sparse.hpp:28-32 (same message)."""
    if s in ("csr", "CSR"):
        return Layout.CSR
    if s in ("csc", "CSC"):
        return Layout.CSC
    raise ValueError(f"unknown layout '{s}' (expected csr or csc)")


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib.spconv_last_error().decode()
    if rc == 1:  # std::invalid_argument in the reference
        raise ValueError(msg)
    raise RuntimeError(msg)  # 2: CUDA / memory, 3: std::runtime_error (I/O, format)


def _ptr(a) -> int:
    """Address of a numpy array or torch tensor (no copies)."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    return getattr(stream, "cuda_stream", stream)


@dataclass(frozen=True)
class ConvSpec:
    """m x n input, k x k kernel, stride s, zero padding p (inc/conv.hpp:33-71)."""
    m: int
    n: int
    k: int
    s: int = 1
    p: int = 0

    def __post_init__(self):
        _check(lib.spconv_spec_check(self.m, self.n, self.k, self.s, self.p))

    @property
    def m_out(self) -> int:
        return (self.m + 2 * self.p - self.k) // self.s + 1

    @property
    def n_out(self) -> int:
        return (self.n + 2 * self.p - self.k) // self.s + 1

    @property
    def input_len(self) -> int:
        return self.m * self.n

    @property
    def output_len(self) -> int:
        return self.m_out * self.n_out

    def str(self) -> str:
        return f"(m={self.m}, n={self.n}, k={self.k}, s={self.s}, p={self.p})"


class Kernel:
    """Dense k x k kernel, row-major, unflipped (inc/conv.hpp:74-96)."""

    def __init__(self, k: int, values: Sequence[float]):
        if k < 1:
            raise ValueError("Kernel: side must be >= 1")
        v = np.asarray(values, dtype=np.float64).reshape(-1)
        if v.size != k * k:
            raise ValueError(f"Kernel: expected {k * k} values, got {v.size}")
        self.k = k
        self.values = v

    def at(self, j: int, i: int) -> float:
        return float(self.values[j * self.k + i])


def nnz_bound(spec: ConvSpec) -> int:
    """Theorem 2.1 total (inc/analysis.hpp:56-66)."""
    out = _i64()
    _check(lib.spconv_nnz_bound(spec.m, spec.n, spec.k, spec.s, spec.p, C.byref(out)))
    return out.value


class Transform:
    """Device-resident T = C*P plus its geometry (inc/conv.hpp:165-168).

    ``spec`` is None for a generic CSR uploaded with :meth:`from_host`."""

    def __init__(self, handle: int, spec: Optional[ConvSpec], device: int):
        self._h = _vp(handle)
        self.spec = spec
        self.device = device
        r, c, z = _i64(), _i64(), _i64()
        _check(lib.spconv_csr_shape(self._h, C.byref(r), C.byref(c), C.byref(z)))
        self.rows, self.cols, self.nnz = r.value, c.value, z.value
        lay = C.c_int()
        _check(lib.spconv_csr_layout(self._h, C.byref(lay)))
        self.layout = lay.value

    @property
    def major_dim(self) -> int:
        return self.cols if self.layout == Layout.CSC else self.rows

    @classmethod
    def from_host(cls, rows: int, cols: int, ptr, idx, val, device: int = 0, stream=None,
                  layout: int = Layout.CSR):
        """Uploads a host matrix (ptr over the major dimension of `layout`)."""
        ptr = np.ascontiguousarray(ptr, np.int64)
        idx = np.ascontiguousarray(idx, np.int64)
        val = np.ascontiguousarray(val, np.float64)
        h = _vp()
        _check(lib.spconv_matrix_from_host(rows, cols, layout, ptr.ctypes.data, idx.ctypes.data,
                                           val.ctypes.data, device, _stream_handle(stream),
                                           C.byref(h)))
        return cls(h.value, None, device)

    @property
    def handle(self) -> int:
        return self._h.value

    def export(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        """ptr(), idx(), val() widened to the reference types (inc/sparse.hpp:128-130),
        in the transform's layout."""
        ptr = np.empty(self.major_dim + 1, np.int64)
        idx = np.empty(max(self.nnz, 1), np.int64)
        val = np.empty(max(self.nnz, 1), np.float64)
        _check(lib.spconv_csr_export(self._h, ptr.ctypes.data, idx.ctypes.data, val.ctypes.data))
        return ptr, idx[: self.nnz], val[: self.nnz]

    def device_ptrs(self) -> Tuple[int, int, int]:
        a, b, c = _vp(), _vp(), _vp()
        _check(lib.spconv_csr_device_ptrs(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def copy_native(self, row_ptr, col_idx, vals, stream=None) -> None:
        """Native int32/int32/fp32 arrays into caller buffers (numpy or torch,
        host or device); synchronous."""
        _check(lib.spconv_csr_copy(self._h, _ptr(row_ptr), _ptr(col_idx), _ptr(vals),
                                   _stream_handle(stream)))

    def write_text(self, transform_header: bool = True) -> bytes:
        """write_transform / write_sparse text (inc/conv.hpp:221-224,
        inc/sparse.hpp:400-406), rendered on the device."""
        n = _i64()
        _check(lib.spconv_csr_write_text(self._h, int(transform_header), None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(n.value, 1))
        _check(lib.spconv_csr_write_text(self._h, int(transform_header), buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    @property
    def storage_bytes(self) -> int:
        """Device bytes of the index / value arrays held (spconv_csr_storage_bytes)."""
        b = _i64()
        _check(lib.spconv_csr_storage_bytes(self._h, C.byref(b)))
        return b.value

    @property
    def last_kernel(self) -> str:
        """Kernel(s) the last apply on this transform launched ("a+b" = two launches)."""
        return lib.spconv_csr_last_kernel(self._h).decode()

    def band_check_status(self) -> Tuple[int, int]:
        """(segments, failed) of the last band check (spconv_band_check_status)."""
        a, b = _i64(), _i64()
        _check(lib.spconv_band_check_status(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def band_check_flags(self) -> np.ndarray:
        """Per-segment verdicts of the last band check (spconv_band_check_flags)."""
        n = _i64()
        _check(lib.spconv_band_check_flags(self._h, None, 0, C.byref(n)))
        out = np.empty(max(n.value, 1), np.uint8)
        _check(lib.spconv_band_check_flags(self._h, out.ctypes.data, out.size, C.byref(n)))
        return out[: n.value]

    def close(self) -> None:
        if self._h and self._h.value:
            lib.spconv_csr_free(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def compile_triplets(rows: int, cols: int, row, col, val, layout: int = Layout.CSR, device: int = 0,
                     stream=None) -> Transform:
    """SparseMatrix::compile(Triplets, layout) (inc/sparse.hpp:35-119) on the
    device: coordinates in any order, duplicates rejected (ValueError with the
    reference's message), explicit zeros kept.  A generic matrix (spec None)."""
    r = np.ascontiguousarray(row, np.int64)
    c = np.ascontiguousarray(col, np.int64)
    v = np.ascontiguousarray(val, np.float64)
    if not (r.size == c.size == v.size):
        raise ValueError("compile_triplets: row, col and val differ in length")
    h = _vp()
    _check(lib.spconv_matrix_from_coo(rows, cols, r.size, r.ctypes.data, c.ctypes.data, v.ctypes.data, layout,
                                      device, _stream_handle(stream), C.byref(h)))
    return Transform(h.value, None, device)


def spgemm(a: Transform, b: Transform, layout: int = Layout.CSR, stream=None) -> Transform:
    """spgemm (inc/sparse.hpp:296-342) on the device, bit-exact in fp64."""
    h = _vp()
    _check(lib.spconv_spgemm(a._h, b._h, layout, _stream_handle(stream), C.byref(h)))
    return Transform(h.value, None, a.device)


def build_padding_matrix(spec: ConvSpec, layout: int = Layout.CSR, device: int = 0, stream=None) -> Transform:
    """P (inc/conv.hpp:125-135), built on the device."""
    h = _vp()
    _check(lib.spconv_build_padding_matrix(spec.m, spec.n, spec.k, spec.s, spec.p, layout, device,
                                           _stream_handle(stream), C.byref(h)))
    return Transform(h.value, None, device)


def build_conv_matrix(kern: Kernel, spec: ConvSpec, layout: int = Layout.CSR, device: int = 0,
                      stream=None) -> Transform:
    """C (inc/conv.hpp:141-162), zero taps stored, built on the device."""
    if kern.k != spec.k:
        raise ValueError(f"build_conv_matrix: kernel side {kern.k} does not match spec {spec.str()}")
    k64 = np.ascontiguousarray(kern.values, np.float64)
    h = _vp()
    _check(lib.spconv_build_conv_matrix(spec.m, spec.n, spec.k, spec.s, spec.p, k64.ctypes.data, layout, device,
                                        _stream_handle(stream), C.byref(h)))
    return Transform(h.value, None, device)


def read_sparse(text: bytes, layout: int = Layout.CSR, device: int = 0, stream=None) -> Transform:
    """read_sparse (inc/sparse.hpp:409-432): a generic matrix (spec None)."""
    if isinstance(text, str):
        text = text.encode()
    h = _vp()
    _check(lib.spconv_sparse_read(text, len(text), layout, device, _stream_handle(stream), C.byref(h)))
    return Transform(h.value, None, device)


def read_transform(text: bytes, device: int = 0, stream=None) -> Transform:
    """read_transform (inc/conv.hpp:226-244): parse, validate, upload (fp32)."""
    if isinstance(text, str):
        text = text.encode()
    h = _vp()
    _check(lib.spconv_transform_read(text, len(text), device, _stream_handle(stream), C.byref(h)))
    spec5 = (C.c_int64 * 5)()
    _check(lib.spconv_csr_spec(h, spec5))
    return Transform(h.value, ConvSpec(*spec5), device)


def format_g17(v: float) -> str:
    """The text writer's "%.17g" of a double (exact; host-callable)."""
    buf = C.create_string_buffer(32)
    n = lib.spconv_format_g17(C.c_double(v), buf)
    return buf.raw[:n].decode()


def build_transform(kern: Kernel, spec: ConvSpec, layout: int = Layout.CSR, device: int = 0,
                    stream=None) -> Transform:
    """On-device build of T in CSR or CSC layout (replaces inc/conv.hpp:179-204;
    both reference routes give the same matrix).  The taps are the reference's
    doubles: entries are kept where the double tap is non-zero, and taps fp32
    cannot represent keep their exact values for export / text / spmm_f64
    (spconv_build_transform_f64); the fp32 kernels apply the narrowed taps."""
    if kern.k != spec.k:
        raise ValueError(f"build_conv_matrix: kernel side {kern.k} does not match spec {spec.str()}")
    k64 = np.ascontiguousarray(kern.values, np.float64)
    h = _vp()
    _check(lib.spconv_build_transform_f64(spec.m, spec.n, spec.k, spec.s, spec.p, k64.ctypes.data,
                                          layout, device, _stream_handle(stream), C.byref(h)))
    return Transform(h.value, spec, device)


def relayout(t: Transform, layout: int, stream=None) -> Transform:
    """relayout (inc/sparse.hpp:268-274): the same matrix in `layout` (new handle)."""
    h = _vp()
    _check(lib.spconv_relayout(t._h, layout, _stream_handle(stream), C.byref(h)))
    return Transform(h.value, t.spec, t.device)


def _dev_f32(t, what):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32):
        raise ValueError(f"{what}: expected a CUDA float32 tensor")
    return t


def spmv(t: Transform, x, y=None, stream=None):
    """y = T x on device (replaces inc/sparse.hpp:214-261); x, y CUDA float32."""
    import torch
    x = _dev_f32(x, "spmv")
    if x.numel() != t.cols:
        raise ValueError(f"spmv: matrix has {t.cols} columns but vector has {x.numel()} elements")
    x = x.contiguous()
    if y is None:
        y = torch.empty(t.rows, dtype=torch.float32, device=x.device)
    _check(lib.spconv_spmv(t._h, x.data_ptr(), y.data_ptr(), _stream_handle(stream)))
    return y


def spmv_group(ts, xs, ys=None, stream=None):
    """ys[i] = ts[i] xs[i] for every member in one launch (spconv_spmv_group):
    a list of transforms, each with its own CUDA vector.  float32 vectors:
    each output bit-identical to spmv(ts[i], xs[i]); float64 vectors: the
    reference's arithmetic (spconv_spmv_group_f64), each output bit-identical
    to spmm_f64 on that member."""
    import torch
    ts, xs = list(ts), list(xs)
    if len(ts) != len(xs):
        raise ValueError("spmv_group: one vector per transform")
    f64 = bool(xs) and xs[0].dtype == torch.float64
    dt = torch.float64 if f64 else torch.float32
    for i, (t, x) in enumerate(zip(ts, xs)):
        if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != dt:
            raise ValueError(f"spmv_group: expected CUDA {dt} vectors (all of one dtype)")
        if x.numel() != t.cols:
            raise ValueError(f"spmv_group: matrix has {t.cols} columns but vector has {x.numel()} elements")
        xs[i] = x.contiguous()
    if ys is None:
        ys = [torch.empty(t.rows, dtype=dt, device=x.device) for t, x in zip(ts, xs)]
    n = len(ts)
    H = np.fromiter((t._h.value for t in ts), np.uintp, n)
    X = np.fromiter((x.data_ptr() for x in xs), np.uintp, n)
    Y = np.fromiter((y.data_ptr() for y in ys), np.uintp, n)
    fn = lib.spconv_spmv_group_f64 if f64 else lib.spconv_spmv_group
    _check(fn(H.ctypes.data, n, X.ctypes.data, Y.ctypes.data, _stream_handle(stream)))
    return ys


def _convolve_group(ts, images, out, dt, fn, who):
    ts = list(ts)
    n = len(ts)
    if len(images) != n:
        raise ValueError(f"{who}: one image per transform")
    cols = np.fromiter((t.cols for t in ts), np.int64, n)
    rows = np.fromiter((t.rows for t in ts), np.int64, n)
    # one packed input (a single C-level copy), members addressed by offset
    packed = np.concatenate([np.ravel(x) for x in images]).astype(dt, copy=False) if n else np.empty(0, dt)
    sizes = np.fromiter((np.size(x) for x in images), np.int64, n)
    if not np.array_equal(sizes, cols):
        i = int(np.nonzero(sizes != cols)[0][0])
        raise ValueError(f"{who}: matrix has {int(cols[i])} columns but image has {int(sizes[i])} elements")
    xoff = np.zeros(n + 1, np.int64)
    np.cumsum(cols, out=xoff[1:])
    off = np.zeros(n + 1, np.int64)
    np.cumsum(rows, out=off[1:])
    if out is None:
        out = np.empty(int(off[-1]), dt)
    elif out.dtype != dt or out.size < off[-1] or not out.flags.c_contiguous:
        raise ValueError(f"{who}: out must be a contiguous {np.dtype(dt).name} array of sum(rows) elements")
    isz = np.dtype(dt).itemsize
    H = np.fromiter((t._h.value for t in ts), np.uintp, n)
    X = packed.__array_interface__["data"][0] + isz * xoff[:-1].astype(np.uintp)
    Y = out.__array_interface__["data"][0] + isz * off[:-1].astype(np.uintp)
    _check(fn(H.ctypes.data, n, X.ctypes.data, Y.ctypes.data))
    return [out[a:b] for a, b in zip(off[:-1].tolist(), off[1:].tolist())]


def convolve_group(ts, images, out=None):
    """Host vectors in, host vectors out (spconv_convolve_host_group, fp32):
    one packed transfer each way and one launch for the whole list.  Returns
    one vector per transform, views into a single output array (``out``, of
    sum(rows) elements, is used when given)."""
    return _convolve_group(ts, images, out, np.float32, lib.spconv_convolve_host_group, "convolve_group")


def convolve_group_f64(ts, images, out=None):
    """convolve_group in the reference's fp64 arithmetic
    (spconv_convolve_host_group_f64): each output bit-identical to the
    reference's convolve() of that layer."""
    return _convolve_group(ts, images, out, np.float64, lib.spconv_convolve_host_group_f64, "convolve_group_f64")


def spmm(t: Transform, X, Y=None, stream=None):
    """Y[b] = T X[b] on device; X [batch, cols] CUDA float32 (row stride = ldx)."""
    import torch
    X = _dev_f32(X, "spmm")
    if X.dim() != 2 or X.shape[1] != t.cols or X.stride(1) != 1:
        raise ValueError(f"spmm: expected X of shape [batch, {t.cols}] with unit column stride")
    if Y is None:
        Y = torch.empty(X.shape[0], t.rows, dtype=torch.float32, device=X.device)
    _check(lib.spconv_spmm(t._h, X.data_ptr(), X.stride(0), Y.data_ptr(), Y.stride(0), X.shape[0],
                           _stream_handle(stream)))
    return Y


def convolve_batch(t: Transform, X_host, Y_host=None):
    """End-to-end apply on HOST fp32 buffers [batch, cols] -> [batch, rows]
    (H2D, SpMM and D2H pipelined inside the library)."""
    if isinstance(X_host, np.ndarray):
        X_host = np.ascontiguousarray(X_host, np.float32)
        batch = X_host.shape[0] if X_host.ndim == 2 else 1
        if Y_host is None:
            Y_host = np.empty((batch, t.rows), np.float32)
    else:  # torch CPU tensor (pinned for full overlap)
        import torch
        assert X_host.device.type == "cpu" and X_host.dtype == torch.float32 and X_host.is_contiguous()
        batch = X_host.shape[0] if X_host.dim() == 2 else 1
        if Y_host is None:
            Y_host = torch.empty(batch, t.rows, dtype=torch.float32, pin_memory=X_host.is_pinned())
    n = X_host.size if isinstance(X_host, np.ndarray) else X_host.numel()
    if n != batch * t.cols:
        raise ValueError(f"convolve_batch: expected {batch}x{t.cols} input values, got {n}")
    _check(lib.spconv_convolve_host(t._h, _ptr(X_host), _ptr(Y_host), batch))
    return Y_host


def convolve_batch_f64(t: Transform, X_host, Y_host=None, threads: int = 1):
    """The reference-semantics apply on HOST fp64 buffers [batch, cols] ->
    [batch, rows] (spconv_convolve_host_f64_threads): bit-identical to the
    reference's convolve() / spmv(m, x, threads) of every image."""
    if isinstance(X_host, np.ndarray):
        X_host = np.ascontiguousarray(X_host, np.float64)
        batch = X_host.shape[0] if X_host.ndim == 2 else 1
        if Y_host is None:
            Y_host = np.empty((batch, t.rows), np.float64)
    else:  # torch CPU tensor
        import torch
        assert X_host.device.type == "cpu" and X_host.dtype == torch.float64 and X_host.is_contiguous()
        batch = X_host.shape[0] if X_host.dim() == 2 else 1
        if Y_host is None:
            Y_host = torch.empty(batch, t.rows, dtype=torch.float64, pin_memory=X_host.is_pinned())
    n = X_host.size if isinstance(X_host, np.ndarray) else X_host.numel()
    if n != batch * t.cols:
        raise ValueError(f"convolve_batch_f64: expected {batch}x{t.cols} input values, got {n}")
    _check(lib.spconv_convolve_host_f64_threads(t._h, _ptr(X_host), _ptr(Y_host), batch, int(threads)))
    return Y_host


def spmm_f64(t: Transform, X, Y=None, stream=None, threads: int = 1):
    """Y[b] = T X[b] in fp64 with the reference's arithmetic (spconv_spmm_f64):
    X [batch, cols] CUDA float64; bit-identical to the reference's spmv(m, x,
    threads) (the handle's exact double values are used when it keeps them;
    `threads` matters for CSC storage only: the reference's per-thread partial
    combine, inc/sparse.hpp:243-258)."""
    import torch
    if not (isinstance(X, torch.Tensor) and X.is_cuda and X.dtype == torch.float64):
        raise ValueError("spmm_f64: expected a CUDA float64 tensor")
    if X.dim() != 2 or X.shape[1] != t.cols or X.stride(1) != 1:
        raise ValueError(f"spmm_f64: expected X of shape [batch, {t.cols}] with unit column stride")
    if Y is None:
        Y = torch.empty(X.shape[0], t.rows, dtype=torch.float64, device=X.device)
    _check(lib.spconv_spmm_f64_threads(t._h, X.data_ptr(), X.stride(0), Y.data_ptr(), Y.stride(0), X.shape[0],
                                       int(threads), _stream_handle(stream)))
    return Y


def convolve(t: Transform, a, threads: int = 1) -> np.ndarray:
    """Reference-semantics apply of one m x n grid (inc/conv.hpp:207-215):
    fp64 in, fp64 device arithmetic with the reference's rounding, fp64 out --
    bit-identical to the reference (exact double taps included)."""
    a = np.asarray(a, dtype=np.float64)
    if t.spec is None:
        raise ValueError("convolve: transform has no geometry (generic CSR)")
    if a.ndim != 2 or a.shape != (t.spec.m, t.spec.n):
        r, c = (a.shape + (1, 1))[:2] if a.ndim >= 1 else (0, 0)
        raise ValueError(f"convolve: input is {r}x{c} but transform expects {t.spec.str()}")
    a = np.ascontiguousarray(a)
    out = np.empty(t.rows, np.float64)
    _check(lib.spconv_convolve_host_f64_threads(t._h, a.ctypes.data, out.ctypes.data, 1, int(threads)))
    return out.reshape(t.spec.m_out, t.spec.n_out)


def direct_conv(spec: ConvSpec, A, taps, out=None, mag=None, stream=None):
    """Device direct_conv (inc/reference.hpp:41-61) of A [batch, m*n] (CUDA
    float32: fmaf contract, or float64: the reference's arithmetic, bit-exact)."""
    import torch
    dt = {torch.float32: 0, torch.float64: 1}[A.dtype]
    A = A.reshape(-1, spec.input_len).contiguous()
    taps = taps.to(device=A.device, dtype=A.dtype).contiguous()
    if out is None:
        out = torch.empty(A.shape[0], spec.output_len, dtype=A.dtype, device=A.device)
    _check(lib.spconv_direct_conv(spec.m, spec.n, spec.k, spec.s, spec.p, dt, taps.data_ptr(), A.data_ptr(),
                                  out.data_ptr(), mag.data_ptr() if mag is not None else None, A.shape[0],
                                  _stream_handle(stream)))
    return out


def im2col_conv(spec: ConvSpec, A, taps, out=None, stream=None):
    """Device im2col lowering + product (inc/reference.hpp:73-136)."""
    import torch
    dt = {torch.float32: 0, torch.float64: 1}[A.dtype]
    A = A.reshape(-1, spec.input_len).contiguous()
    taps = taps.to(device=A.device, dtype=A.dtype).contiguous()
    if out is None:
        out = torch.empty(A.shape[0], spec.output_len, dtype=A.dtype, device=A.device)
    patches = torch.empty(A.shape[0] * spec.k * spec.k * spec.output_len, dtype=A.dtype, device=A.device)
    _check(lib.spconv_im2col_conv(spec.m, spec.n, spec.k, spec.s, spec.p, dt, taps.data_ptr(), A.data_ptr(),
                                  out.data_ptr(), patches.data_ptr(), A.shape[0], _stream_handle(stream)))
    return out


def run_verification(max_dim: int = 12, seeds: int = 3, base_seed: int = 42, device: int = 0) -> dict:
    """run_verification (inc/verify.hpp:59-169) over the device path (see
    include/spconv_b200.h); returns the VerifyReport fields."""
    counts = (C.c_int64 * 4)()
    devs = (C.c_double * 3)()
    buf = C.create_string_buffer(8192)
    _check(lib.spconv_run_verification(max_dim, seeds, base_seed, device, counts, devs, buf, len(buf)))
    fails = [f for f in buf.value.decode().split("\n") if f]
    return dict(specs=counts[0], conv_cases=counts[1], clipped_specs=counts[2], failures=counts[3],
                max_conv_dev=devs[0], max_layout_dev=devs[1], max_rel_dev=devs[2], failure_lines=fails)
