"""TEST INFRASTRUCTURE ONLY -- the parity checkers for the conv-as-SpMV path.

Two ctypes front-ends over C libraries built by ``oracle/Makefile``:

* :class:`Oracle` -- ``_build/libspconv_oracle.so``, the plain-C restatement in
  ``spconv_oracle.c`` (every function cites the reference file:line it follows).
* :class:`Ref` -- ``_ref/libspconv_ref.so``, the reference's own headers
  (``/root/reference/proj/include/spconv``) compiled unmodified behind the
  extern "C" shim ``ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product (``paper_2411_19419_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libspconv_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspconv_ref.so")

i64 = C.c_int64
u64 = C.c_uint64
PI64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
PF64 = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
PF32 = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    """The C restatement (``spconv_oracle.c``)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        L = C.CDLL(path)
        L.orc_derive_seed.restype = u64
        L.orc_derive_seed.argtypes = [u64, u64]
        L.orc_random_normal.argtypes = [u64, i64, C.c_void_p]
        L.orc_random_normal_f32.argtypes = [u64, i64, C.c_void_p]
        L.orc_spec_check.argtypes = [i64] * 5
        L.orc_nnz_bound.restype = i64
        L.orc_nnz_bound.argtypes = [i64] * 5
        L.orc_nnz_oracle.restype = i64
        L.orc_nnz_oracle.argtypes = [i64] * 5
        L.orc_nnz_per_output.argtypes = [i64] * 5 + [C.c_void_p]
        L.orc_build_transform.restype = i64
        L.orc_build_transform.argtypes = [i64] * 5 + [C.c_void_p] * 4
        L.orc_spmv_csr_f64.argtypes = [i64] + [C.c_void_p] * 5
        L.orc_spmv_csr_f32_fma.argtypes = [i64] + [C.c_void_p] * 5
        L.orc_spmm_csr_f32_fma.argtypes = [i64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, i64,
                                           C.c_void_p, i64, i64]
        L.orc_build_transform_native.restype = i64
        L.orc_build_transform_native.argtypes = [i64] * 5 + [C.c_void_p] * 4
        L.orc_spmm_native_f32_fma.argtypes = [i64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              i64, C.c_void_p, i64, i64]
        L.orc_spmv_abs_f64.argtypes = [i64] + [C.c_void_p] * 5
        L.orc_direct_conv.argtypes = [i64] * 5 + [C.c_void_p] * 3
        L.orc_transpose.argtypes = [i64, i64] + [C.c_void_p] * 6
        L.orc_spmv_csc_f64.argtypes = [i64] + [C.c_void_p] * 5 + [i64]
        L.orc_spmv_csc_f32_fma.argtypes = [i64] + [C.c_void_p] * 5 + [i64]
        L.orc_spmv_csc_f64_threads.argtypes = [i64] + [C.c_void_p] * 5 + [i64, i64]
        self.L = L

    # -- rng.hpp ------------------------------------------------------------
    def derive_seed(self, base: int, index: int) -> int:
        return int(self.L.orc_derive_seed(base, index))

    def random_normal(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.float64)
        self.L.orc_random_normal(seed, count, _p(out))
        return out

    def random_normal_f32(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.float32)
        self.L.orc_random_normal_f32(seed, count, _p(out))
        return out

    # -- conv.hpp / analysis.hpp -------------------------------------------
    def spec_check(self, m, n, k, s, p) -> int:
        return int(self.L.orc_spec_check(m, n, k, s, p))

    def nnz_bound(self, m, n, k, s, p) -> int:
        return int(self.L.orc_nnz_bound(m, n, k, s, p))

    def nnz_oracle(self, m, n, k, s, p) -> int:
        return int(self.L.orc_nnz_oracle(m, n, k, s, p))

    def nnz_per_output(self, m, n, k, s, p) -> np.ndarray:
        mo, no = (m + 2 * p - k) // s + 1, (n + 2 * p - k) // s + 1
        out = np.empty(mo * no, np.int64)
        self.L.orc_nnz_per_output(m, n, k, s, p, _p(out))
        return out

    def build_transform(self, m, n, k, s, p, kern) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        kern = np.ascontiguousarray(kern, np.float64).reshape(-1)
        assert kern.size == k * k
        nnz = int(self.L.orc_build_transform(m, n, k, s, p, _p(kern), None, None, None))
        if nnz < 0:
            raise ValueError(f"invalid spec {(m, n, k, s, p)}")
        mo, no = (m + 2 * p - k) // s + 1, (n + 2 * p - k) // s + 1
        ptr = np.empty(mo * no + 1, np.int64)
        idx = np.empty(max(nnz, 1), np.int64)
        val = np.empty(max(nnz, 1), np.float64)
        self.L.orc_build_transform(m, n, k, s, p, _p(kern), _p(ptr), _p(idx), _p(val))
        return ptr, idx[:nnz], val[:nnz]

    def build_native(self, m, n, k, s, p, kern32):
        """Same CSR in the device format: int32 ptr/idx, fp32 val."""
        kern32 = np.ascontiguousarray(kern32, np.float32).reshape(-1)
        nnz = int(self.L.orc_build_transform_native(m, n, k, s, p, _p(kern32), None, None, None))
        if nnz < 0:
            raise ValueError(f"invalid spec {(m, n, k, s, p)}")
        mo, no = (m + 2 * p - k) // s + 1, (n + 2 * p - k) // s + 1
        ptr = np.empty(mo * no + 1, np.int32)
        idx = np.empty(max(nnz, 1), np.int32)
        val = np.empty(max(nnz, 1), np.float32)
        self.L.orc_build_transform_native(m, n, k, s, p, _p(kern32), _p(ptr), _p(idx), _p(val))
        return ptr, idx[:nnz], val[:nnz]

    def spmm_native(self, ptr, idx, val, X) -> np.ndarray:
        """Ordered-fmaf fp32 SpMM over the native format; X [batch, cols] f32."""
        X = np.ascontiguousarray(X, np.float32)
        if X.ndim == 1:
            X = X[None]
        rows = ptr.size - 1
        Y = np.empty((X.shape[0], rows), np.float32)
        self.L.orc_spmm_native_f32_fma(rows, _p(ptr), _p(idx), _p(val), _p(X), X.shape[1], _p(Y),
                                       rows, X.shape[0])
        return Y

    # -- sparse.hpp ---------------------------------------------------------
    def spmv_f64(self, ptr, idx, val, x) -> np.ndarray:
        rows = ptr.size - 1
        y = np.empty(rows, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        self.L.orc_spmv_csr_f64(rows, _p(ptr), _p(idx), _p(np.ascontiguousarray(val, np.float64)),
                                _p(x), _p(y))
        return y

    def spmv_f32_fma(self, ptr, idx, val, x) -> np.ndarray:
        rows = ptr.size - 1
        y = np.empty(rows, np.float32)
        x = np.ascontiguousarray(x, np.float32)
        self.L.orc_spmv_csr_f32_fma(rows, _p(ptr), _p(idx),
                                    _p(np.ascontiguousarray(val, np.float32)), _p(x), _p(y))
        return y

    def spmm_f32_fma(self, ptr, idx, val, X) -> np.ndarray:
        """X: [batch, cols] float32 image-major -> Y: [batch, rows]."""
        X = np.ascontiguousarray(X, np.float32)
        rows = ptr.size - 1
        Y = np.empty((X.shape[0], rows), np.float32)
        self.L.orc_spmm_csr_f32_fma(rows, _p(ptr), _p(idx), _p(np.ascontiguousarray(val, np.float32)),
                                    _p(X), X.shape[1], _p(Y), rows, X.shape[0])
        return Y

    def spmv_abs(self, ptr, idx, val, x) -> np.ndarray:
        rows = ptr.size - 1
        y = np.empty(rows, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        self.L.orc_spmv_abs_f64(rows, _p(ptr), _p(idx), _p(np.ascontiguousarray(val, np.float64)),
                                _p(x), _p(y))
        return y

    def transpose(self, major, minor, ptr, idx, val):
        """relayout (inc/sparse.hpp:268-274): the storage of the other layout."""
        ptr = np.ascontiguousarray(ptr, np.int64)
        idx = np.ascontiguousarray(idx, np.int64)
        val = np.ascontiguousarray(val, np.float64)
        nnz = int(ptr[major])
        optr = np.empty(minor + 1, np.int64)
        oidx = np.empty(max(nnz, 1), np.int64)
        oval = np.empty(max(nnz, 1), np.float64)
        self.L.orc_transpose(major, minor, _p(ptr), _p(idx), _p(val), _p(optr), _p(oidx), _p(oval))
        return optr, oidx[:nnz], oval[:nnz]

    def spmv_csc_f64(self, rows, ptr, idx, val, x) -> np.ndarray:
        cols = ptr.size - 1
        y = np.empty(rows, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        self.L.orc_spmv_csc_f64(cols, _p(np.ascontiguousarray(ptr, np.int64)),
                                _p(np.ascontiguousarray(idx, np.int64)),
                                _p(np.ascontiguousarray(val, np.float64)), _p(x), _p(y), rows)
        return y

    def spmv_csc_f64_threads(self, rows, ptr, idx, val, x, threads) -> np.ndarray:
        cols = ptr.size - 1
        y = np.empty(rows, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        self.L.orc_spmv_csc_f64_threads(cols, _p(np.ascontiguousarray(ptr, np.int64)),
                                        _p(np.ascontiguousarray(idx, np.int64)),
                                        _p(np.ascontiguousarray(val, np.float64)), _p(x), _p(y), rows, threads)
        return y

    def spmv_csc_f32_fma(self, rows, ptr, idx, val, x) -> np.ndarray:
        cols = ptr.size - 1
        y = np.empty(rows, np.float32)
        x = np.ascontiguousarray(x, np.float32)
        self.L.orc_spmv_csc_f32_fma(cols, _p(np.ascontiguousarray(ptr, np.int64)),
                                    _p(np.ascontiguousarray(idx, np.int64)),
                                    _p(np.ascontiguousarray(val, np.float32)), _p(x), _p(y), rows)
        return y

    def direct_conv(self, m, n, k, s, p, a, kern) -> np.ndarray:
        mo, no = (m + 2 * p - k) // s + 1, (n + 2 * p - k) // s + 1
        out = np.empty(mo * no, np.float64)
        a = np.ascontiguousarray(a, np.float64)
        kern = np.ascontiguousarray(kern, np.float64)
        if self.L.orc_direct_conv(m, n, k, s, p, _p(a), _p(kern), _p(out)) != 0:
            raise ValueError("invalid spec")
        return out


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Ref:
    """The reference headers compiled as-is (``oracle/_ref/libspconv_ref.so``)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference library missing: {path}")
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_derive_seed.restype = u64
        L.ref_derive_seed.argtypes = [u64, u64]
        L.ref_random_normal_grid.argtypes = [i64, i64, u64, C.c_void_p]
        L.ref_random_normal_kernel.argtypes = [i64, u64, C.c_void_p]
        L.ref_spec_check.argtypes = [i64] * 5
        L.ref_nnz_bound.argtypes = [i64] * 5 + [C.c_void_p]
        L.ref_nnz_oracle.argtypes = [i64] * 5 + [C.c_void_p]
        L.ref_nnz_per_output.argtypes = [i64] * 5 + [C.c_void_p]
        L.ref_build_transform.argtypes = [i64] * 5 + [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_transform_shape.argtypes = [C.c_void_p] + [C.POINTER(i64)] * 3
        L.ref_transform_export.argtypes = [C.c_void_p] * 4
        L.ref_convolve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, i64, C.c_int]
        L.ref_transform_free.argtypes = [C.c_void_p]
        L.ref_direct_conv.argtypes = [i64] * 5 + [C.c_void_p] * 3
        L.ref_run_verification.argtypes = [i64, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_hardware_concurrency.restype = C.c_uint
        if hasattr(L, "ref_write_transform"):
            L.ref_write_transform.argtypes = [C.c_void_p, C.c_void_p, i64, C.POINTER(i64)]
            L.ref_write_sparse_csr.argtypes = [i64, i64] + [C.c_void_p] * 4 + [i64, C.POINTER(i64)]
            L.ref_read_transform.argtypes = [C.c_char_p, i64, C.POINTER(C.c_void_p)]
        L.ref_build_transform_layout.argtypes = [i64] * 5 + [C.c_void_p, C.c_int, C.c_int,
                                                              C.POINTER(C.c_void_p)]
        L.ref_relayout.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_transform_layout.argtypes = [C.c_void_p]
        if hasattr(L, "ref_run_layer_bench"):
            L.ref_run_layer_bench.argtypes = [C.c_char_p] + [i64] * 7 + [u64, C.c_int, C.c_void_p]
        self.L = L

    def _chk(self, rc: int):
        if rc != 0:
            raise RefError(rc, self.L.ref_last_error().decode())

    def derive_seed(self, base, index) -> int:
        return int(self.L.ref_derive_seed(base, index))

    def random_normal_grid(self, rows, cols, seed) -> np.ndarray:
        out = np.empty(rows * cols, np.float64)
        self._chk(self.L.ref_random_normal_grid(rows, cols, seed, _p(out)))
        return out

    def random_normal_kernel(self, k, seed) -> np.ndarray:
        out = np.empty(k * k, np.float64)
        self._chk(self.L.ref_random_normal_kernel(k, seed, _p(out)))
        return out

    def spec_check(self, m, n, k, s, p):
        self._chk(self.L.ref_spec_check(m, n, k, s, p))

    def nnz_bound(self, m, n, k, s, p) -> int:
        v = np.zeros(1, np.int64)
        self._chk(self.L.ref_nnz_bound(m, n, k, s, p, _p(v)))
        return int(v[0])

    def nnz_oracle(self, m, n, k, s, p) -> int:
        v = np.zeros(1, np.int64)
        self._chk(self.L.ref_nnz_oracle(m, n, k, s, p, _p(v)))
        return int(v[0])

    def nnz_per_output(self, m, n, k, s, p) -> np.ndarray:
        mo, no = (m + 2 * p - k) // s + 1, (n + 2 * p - k) // s + 1
        out = np.empty(mo * no, np.int64)
        self._chk(self.L.ref_nnz_per_output(m, n, k, s, p, _p(out)))
        return out

    def build(self, m, n, k, s, p, kern, route: int = 0, layout: int = 0) -> "RefTransform":
        """build_transform (inc/conv.hpp:179-204); layout 0 = CSR, 1 = CSC."""
        kern = np.ascontiguousarray(kern, np.float64).reshape(-1)
        h = C.c_void_p()
        if layout:
            self._chk(self.L.ref_build_transform_layout(m, n, k, s, p, _p(kern), route, layout, C.byref(h)))
        else:
            self._chk(self.L.ref_build_transform(m, n, k, s, p, _p(kern), route, C.byref(h)))
        return RefTransform(self, h, (m, n, k, s, p))

    def direct_conv(self, m, n, k, s, p, a, kern) -> np.ndarray:
        mo, no = (m + 2 * p - k) // s + 1, (n + 2 * p - k) // s + 1
        out = np.empty(mo * no, np.float64)
        self._chk(self.L.ref_direct_conv(m, n, k, s, p, _p(np.ascontiguousarray(a, np.float64)),
                                         _p(np.ascontiguousarray(kern, np.float64)), _p(out)))
        return out

    def run_verification(self, max_dim=12, seeds=3):
        out4 = np.zeros(4, np.int64)
        dev2 = np.zeros(2, np.float64)
        self._chk(self.L.ref_run_verification(max_dim, seeds, _p(out4), _p(dev2)))
        return dict(specs=int(out4[0]), conv_cases=int(out4[1]), clipped_specs=int(out4[2]),
                    failures=int(out4[3]), max_conv_dev=float(dev2[0]), max_layout_dev=float(dev2[1]))

    def hardware_concurrency(self) -> int:
        return int(self.L.ref_hardware_concurrency())

    def write_sparse_csr(self, rows, cols, ptr, idx, val) -> bytes:
        """write_sparse (inc/sparse.hpp:400-406) of the CSR (ptr, idx, val)."""
        ptr = np.ascontiguousarray(ptr, np.int64)
        idx = np.ascontiguousarray(idx, np.int64)
        val = np.ascontiguousarray(val, np.float64)
        n = i64()
        self._chk(self.L.ref_write_sparse_csr(rows, cols, _p(ptr), _p(idx), _p(val), None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(n.value, 1))
        self._chk(self.L.ref_write_sparse_csr(rows, cols, _p(ptr), _p(idx), _p(val), buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def read_transform(self, text: bytes) -> "RefTransform":
        h = C.c_void_p()
        self._chk(self.L.ref_read_transform(text, len(text), C.byref(h)))
        t = RefTransform(self, h, None)
        return t

    def run_layer_bench(self, name, m, n, k, s, p, trials, warmup, seed, threads=1):
        """inc/bench.hpp:202-261 on one layer -> {method: (mean_us, sem_us, build_us)}."""
        out = np.zeros(9, np.float64)
        self._chk(self.L.ref_run_layer_bench(name.encode(), m, n, k, s, p, trials, warmup, seed,
                                             threads, _p(out)))
        return {meth: tuple(out[3 * i: 3 * i + 3]) for i, meth in
                enumerate(("CSR-SpMV", "CSC-SpMV", "im2col"))}


class RefTransform:
    def __init__(self, ref: Ref, h, spec):
        self.ref, self.h, self.spec = ref, h, spec

    @property
    def layout(self) -> int:
        return int(self.ref.L.ref_transform_layout(self.h))

    def relayout(self, layout: int) -> "RefTransform":
        """relayout (inc/sparse.hpp:268-274) of the matrix, same spec."""
        h = C.c_void_p()
        self.ref._chk(self.ref.L.ref_relayout(self.h, layout, C.byref(h)))
        return RefTransform(self.ref, h, self.spec)

    def shape(self):
        r, c, z = i64(), i64(), i64()
        self.ref.L.ref_transform_shape(self.h, C.byref(r), C.byref(c), C.byref(z))
        return r.value, c.value, z.value

    def export(self):
        """(ptr, idx, val) in the matrix's own layout (ptr over the major dim)."""
        rows, cols, nnz = self.shape()
        ptr = np.empty((cols if self.layout else rows) + 1, np.int64)
        idx = np.empty(max(nnz, 1), np.int64)
        val = np.empty(max(nnz, 1), np.float64)
        self.ref.L.ref_transform_export(self.h, _p(ptr), _p(idx), _p(val))
        return ptr, idx[:nnz], val[:nnz]

    def write_text(self) -> bytes:
        """write_transform (inc/conv.hpp:221-224)."""
        n = i64()
        self.ref._chk(self.ref.L.ref_write_transform(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(n.value, 1))
        self.ref._chk(self.ref.L.ref_write_transform(self.h, buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def convolve(self, X: np.ndarray, threads: int = 1) -> np.ndarray:
        """X: [batch, m*n] float64 -> [batch, m_out*n_out] float64 (reference convolve)."""
        X = np.ascontiguousarray(X, np.float64)
        if X.ndim == 1:
            X = X[None]
        rows, _, _ = self.shape()
        Y = np.empty((X.shape[0], rows), np.float64)
        self.ref._chk(self.ref.L.ref_convolve(self.h, _p(X), _p(Y), X.shape[0], threads))
        return Y

    def close(self):
        if self.h:
            self.ref.L.ref_transform_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def try_ref() -> Optional[Ref]:
    """The compiled reference, or None when oracle/_ref was never built."""
    try:
        return Ref()
    except (FileNotFoundError, OSError):
        return None
