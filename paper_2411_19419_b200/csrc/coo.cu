// coo.cu -- SparseMatrix::compile(Triplets, layout) on the device
// (inc/sparse.hpp:35-119): coordinate entries in insertion order -> compressed
// storage in (major, minor) order, duplicates rejected with the reference's
// message, explicit zeros kept.
//
//   key = major * minor_dim + minor (64-bit), a stable CUB radix sort of
//   (key, insertion index); a duplicate is two equal neighbouring keys (the
//   first one in sorted order is reported, as compile() reports it); ptr comes
//   from the key boundaries (each element fills the ptr slots of the empty
//   majors before it), idx = key % minor_dim, values gathered through the
//   permutation (fp32 narrowed, fp64 kept when the caller asks).
#include <algorithm>

#include <cub/cub.cuh>

#include "internal.h"

namespace spb {

namespace {

__global__ void coo_keys(long long n, const int64_t* r, const int64_t* c, int64_t minor_dim, bool by_row,
                         unsigned long long* key, int* perm) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int64_t major = by_row ? r[i] : c[i], minor = by_row ? c[i] : r[i];
        key[i] = (unsigned long long)(major * minor_dim + minor);
        perm[i] = (int)i;
    }
}

__global__ void coo_first_dup(long long n, const unsigned long long* key, unsigned long long* first) {
    for (long long i = 1 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        if (key[i] == key[i - 1]) atomicMin(first, (unsigned long long)i);
}

__global__ void coo_fill(long long n, const unsigned long long* key, const int* perm, const double* val,
                         int64_t minor_dim, int64_t major_dim, int32_t* ptr, int32_t* idx, float* v32, double* v64,
                         int* max_len) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long major = (long long)(key[i] / (unsigned long long)minor_dim);
        idx[i] = (int32_t)(key[i] - (unsigned long long)major * (unsigned long long)minor_dim);
        const double v = val[perm[i]];
        v32[i] = (float)v;
        if (v64) v64[i] = v;
        // ptr[m] = i for every major m in (major(i - 1), major(i)]
        const long long prev = i ? (long long)(key[i - 1] / (unsigned long long)minor_dim) : -1;
        for (long long m = prev + 1; m <= major; ++m) ptr[m] = (int32_t)i;
        if (i == n - 1)
            for (long long m = major + 1; m <= major_dim; ++m) ptr[m] = (int32_t)n;
        // longest major slice: the run that starts here
        if (major != prev) {
            long long lo = i, hi = n;  // first index with a larger major (keys are sorted)
            const unsigned long long lim = (unsigned long long)(major + 1) * (unsigned long long)minor_dim;
            while (lo < hi) {
                const long long mid = (lo + hi) / 2;
                if (key[mid] < lim) lo = mid + 1;
                else hi = mid;
            }
            atomicMax(max_len, (int)(lo - i));
        }
    }
}

__global__ void zero_ptr(int32_t* ptr, long long count) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
        ptr[i] = 0;
}

}  // namespace

// Device compile of n host triplets (already range-checked) into the
// compressed arrays ptr[major_dim + 1], idx[n], v32[n] (and v64[n] when
// non-null), all device buffers; by_row: CSR order.  *dup_index = the sorted
// position of the first duplicate (-1: none), *dup_r / *dup_c its coordinates;
// *max_len = the longest major slice.  Synchronous.
cudaError_t coo_compile(long long n, const int64_t* r_host, const int64_t* c_host, const double* v_host,
                        int64_t rows, int64_t cols, bool by_row, int32_t* ptr, int32_t* idx, float* v32,
                        double* v64, long long* dup_index, int64_t* dup_r, int64_t* dup_c, int* max_len,
                        cudaStream_t st) {
    const int64_t major_dim = by_row ? rows : cols, minor_dim = by_row ? cols : rows;
    *dup_index = -1;
    *max_len = 0;
    if (n == 0) {
        zero_ptr<<<(unsigned)std::min<long long>((major_dim + 256) / 256, 4096), 256, 0, st>>>(ptr, major_dim + 1);
        cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
    }
    // device scratch: r, c, v, keys in/out, perm in/out, counters, CUB temp
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (int*)nullptr, (int*)nullptr, (int)n, 0, 64, st);
    auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t b_rc = up((size_t)n * 8), b_key = up((size_t)n * 8), b_perm = up((size_t)n * 4);
    const size_t total = 3 * b_rc + 2 * b_key + 2 * b_perm + 256 + up(tmp_bytes);
    char* mem = nullptr;
    cudaError_t e = cudaMallocAsync(&mem, total, st);
    if (e != cudaSuccess) return e;
    int64_t* dr = reinterpret_cast<int64_t*>(mem);
    int64_t* dc = reinterpret_cast<int64_t*>(mem + b_rc);
    double* dv = reinterpret_cast<double*>(mem + 2 * b_rc);
    unsigned long long* k0 = reinterpret_cast<unsigned long long*>(mem + 3 * b_rc);
    unsigned long long* k1 = reinterpret_cast<unsigned long long*>(mem + 3 * b_rc + b_key);
    int* p0 = reinterpret_cast<int*>(mem + 3 * b_rc + 2 * b_key);
    int* p1 = reinterpret_cast<int*>(mem + 3 * b_rc + 2 * b_key + b_perm);
    unsigned long long* first = reinterpret_cast<unsigned long long*>(mem + 3 * b_rc + 2 * b_key + 2 * b_perm);
    int* dmax = reinterpret_cast<int*>(first + 1);
    void* tmp = mem + 3 * b_rc + 2 * b_key + 2 * b_perm + 256;
    const unsigned grid = (unsigned)std::min<long long>((n + 255) / 256, 148 * 8);
    // key bits: enough for major_dim * minor_dim
    int bits = 1;
    while (bits < 64 && (1ull << bits) < (unsigned long long)(major_dim * minor_dim)) ++bits;
    unsigned long long init_first = ~0ull;
    int zero = 0;
    e = cudaMemcpyAsync(dr, r_host, (size_t)n * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dc, c_host, (size_t)n * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dv, v_host, (size_t)n * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(first, &init_first, 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dmax, &zero, 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        coo_keys<<<grid, 256, 0, st>>>(n, dr, dc, minor_dim, by_row, k0, p0);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, p0, p1, (int)n, 0, bits, st);
    if (e == cudaSuccess) {
        coo_first_dup<<<grid, 256, 0, st>>>(n, k1, first);
        e = cudaGetLastError();
    }
    unsigned long long fd = ~0ull;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&fd, first, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess && fd != ~0ull) {
        unsigned long long kd = 0;
        e = cudaMemcpy(&kd, k1 + fd, 8, cudaMemcpyDeviceToHost);
        const int64_t maj = (int64_t)(kd / (unsigned long long)minor_dim), mnr = (int64_t)(kd % (unsigned long long)minor_dim);
        *dup_index = (long long)fd;
        *dup_r = by_row ? maj : mnr;
        *dup_c = by_row ? mnr : maj;
    }
    if (e == cudaSuccess && fd == ~0ull) {
        coo_fill<<<grid, 256, 0, st>>>(n, k1, p1, dv, minor_dim, major_dim, ptr, idx, v32, v64, dmax);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpyAsync(max_len, dmax, 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    }
    cudaFreeAsync(mem, st);
    const cudaError_t e2 = cudaStreamSynchronize(st);
    return e != cudaSuccess ? e : e2;
}

}  // namespace spb

namespace spb {

// ---------------------------------------------------------------------------
// spgemm (inc/sparse.hpp:296-342) and the reference's two factor matrices
// (build_padding_matrix / build_conv_matrix, inc/conv.hpp:125-162) on the
// device.
//
// spgemm: every product a_ik * b_kj is expanded in the reference's order (A's
// row entries ascending, then B's row k ascending), keyed by (i, j), and
// stable-sorted by key; each key's run is then summed by one thread in that
// order starting from 0.0 (acc = 0.0; acc += av * bv, one rounded multiply
// and one rounded add each, inc/sparse.hpp:331) -- the reference's sum bit for
// bit -- and kept unless it is exactly 0.0 (:335).
// ---------------------------------------------------------------------------
namespace {

__global__ void row_of_entry(int rows, const int32_t* ptr, int* rowof) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
        for (int e = ptr[r]; e < ptr[r + 1]; ++e) rowof[e] = r;
}

__global__ void product_counts(long long na, const int32_t* aidx, const int32_t* bptr, long long* cnt) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < na; e += (long long)gridDim.x * blockDim.x) {
        const int k = aidx[e];
        cnt[e] = bptr[k + 1] - bptr[k];
    }
}

__device__ __forceinline__ double val64(const float* v32, const double* v64, long long e) {
    return v64 ? v64[e] : (double)v32[e];
}

__global__ void expand_products(long long na, const int* rowof, const int32_t* aidx, const float* av32,
                                const double* av64, const int32_t* bptr, const int32_t* bidx, const float* bv32,
                                const double* bv64, const long long* off, long long ncols, unsigned long long* key,
                                double* prod) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < na; e += (long long)gridDim.x * blockDim.x) {
        const int k = aidx[e];
        const double a = val64(av32, av64, e);
        long long o = off[e];
        for (int q = bptr[k]; q < bptr[k + 1]; ++q, ++o) {
            key[o] = (unsigned long long)rowof[e] * (unsigned long long)ncols + (unsigned long long)bidx[q];
            prod[o] = __dmul_rn(a, val64(bv32, bv64, q));
        }
    }
}

// Runs of equal keys: the thread at a run's start sums it in order; kept[p] =
// 1 at a kept run's start.
__global__ void sum_runs(long long nf, const unsigned long long* key, const double* prod, double* acc_out,
                         int* kept) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < nf; p += (long long)gridDim.x * blockDim.x) {
        int k = 0;
        if (p == 0 || key[p] != key[p - 1]) {
            double acc = 0.0;
            for (long long q = p; q < nf && key[q] == key[p]; ++q) acc = __dadd_rn(acc, prod[q]);
            acc_out[p] = acc;
            k = acc != 0.0 ? 1 : 0;  // (NaN != 0.0: kept)
        }
        kept[p] = k;
    }
}

__global__ void emit_kept(long long nf, const unsigned long long* key, const double* acc, const int* kept,
                          const int* pos, long long ncols, unsigned long long* okey, double* oval) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < nf; p += (long long)gridDim.x * blockDim.x)
        if (kept[p]) {
            okey[pos[p]] = key[p];
            oval[pos[p]] = acc[p];
        }
    (void)ncols;
}

// Compressed arrays from (row * ncols + col)-sorted keys: ptr, idx, fp32 and
// (when v64) fp64 values; *max_len = the longest row.
__global__ void fill_from_keys(long long n, const unsigned long long* key, const double* val, long long ncols,
                               long long nrows, int32_t* ptr, int32_t* idx, float* v32, double* v64, int* max_len) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long row = (long long)(key[i] / (unsigned long long)ncols);
        idx[i] = (int32_t)(key[i] - (unsigned long long)row * (unsigned long long)ncols);
        v32[i] = (float)val[i];
        if (v64) v64[i] = val[i];
        const long long prev = i ? (long long)(key[i - 1] / (unsigned long long)ncols) : -1;
        for (long long m = prev + 1; m <= row; ++m) ptr[m] = (int32_t)i;
        if (i == n - 1)
            for (long long m = row + 1; m <= nrows; ++m) ptr[m] = (int32_t)n;
        if (row != prev) {
            long long lo = i, hi = n;
            const unsigned long long lim = (unsigned long long)(row + 1) * (unsigned long long)ncols;
            while (lo < hi) {
                const long long mid = (lo + hi) / 2;
                if (key[mid] < lim) lo = mid + 1;
                else hi = mid;
            }
            atomicMax(max_len, (int)(lo - i));
        }
    }
}

__global__ void any_inexact(long long n, const double* v, int* flag) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (__double_as_longlong((double)(float)v[i]) != __double_as_longlong(v[i])) *flag = 1;
}

unsigned grid_for(long long n) { return (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 8)); }

}  // namespace

cudaError_t spgemm_device(const SpgemmIn& A, const SpgemmIn& B, SpgemmOut* out, cudaStream_t st) {
    const long long na = A.nnz, ncols = B.cols;
    out->nnz = 0;
    out->max_len = 0;
    out->vals_buf = nullptr;
    out->keys_buf = nullptr;
    out->mem = nullptr;
    if (na == 0) return cudaSuccess;
    auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
    // phase 1: products per A entry, offsets
    char* m1 = nullptr;
    size_t scan_tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (long long*)nullptr, (long long*)nullptr, (int)na, st);
    const size_t b_cnt = up((size_t)(na + 1) * 8), b_row = up((size_t)na * 4);
    cudaError_t e = cudaMallocAsync(&m1, 2 * b_cnt + b_row + up(scan_tmp), st);
    if (e != cudaSuccess) return e;
    long long* cnt = reinterpret_cast<long long*>(m1);
    long long* off = reinterpret_cast<long long*>(m1 + b_cnt);
    int* rowof = reinterpret_cast<int*>(m1 + 2 * b_cnt);
    void* stmp = m1 + 2 * b_cnt + b_row;
    row_of_entry<<<grid_for(A.rows), 256, 0, st>>>(A.rows, A.ptr, rowof);
    product_counts<<<grid_for(na), 256, 0, st>>>(na, A.idx, B.ptr, cnt);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(stmp, scan_tmp, cnt, off, (int)na, st);
    long long last_off = 0, last_cnt = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&last_off, off + na - 1, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&last_cnt, cnt + na - 1, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    const long long nf = last_off + last_cnt;
    if (e != cudaSuccess || nf == 0) {
        cudaFreeAsync(m1, st);
        return e;
    }
    if (nf >= (1ll << 31)) {
        cudaFreeAsync(m1, st);
        return cudaErrorInvalidValue;  // more products than one sort handles
    }
    // phase 2: expand, stable sort by (i, j), sum runs in order, compact
    size_t sort_tmp = 0, sum_tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (double*)nullptr, (double*)nullptr, (int)nf, 0, 64, st);
    cub::DeviceScan::ExclusiveSum(nullptr, sum_tmp, (int*)nullptr, (int*)nullptr, (int)nf, st);
    const size_t b_k = up((size_t)nf * 8), b_i = up((size_t)nf * 4);
    char* m2 = nullptr;
    e = cudaMallocAsync(&m2, 5 * b_k + 2 * b_i + up(std::max(sort_tmp, sum_tmp)) + 256, st);
    if (e != cudaSuccess) {
        cudaFreeAsync(m1, st);
        return e;
    }
    unsigned long long* k0 = reinterpret_cast<unsigned long long*>(m2);
    unsigned long long* k1 = reinterpret_cast<unsigned long long*>(m2 + b_k);
    double* p0 = reinterpret_cast<double*>(m2 + 2 * b_k);
    double* p1 = reinterpret_cast<double*>(m2 + 3 * b_k);
    double* accs = reinterpret_cast<double*>(m2 + 4 * b_k);
    int* kept = reinterpret_cast<int*>(m2 + 5 * b_k);
    int* pos = reinterpret_cast<int*>(m2 + 5 * b_k + b_i);
    void* tmp2 = m2 + 5 * b_k + 2 * b_i;
    int bits = 1;
    while (bits < 64 && (1ull << bits) < (unsigned long long)A.rows * (unsigned long long)ncols) ++bits;
    expand_products<<<grid_for(na), 256, 0, st>>>(na, rowof, A.idx, A.v32, A.v64, B.ptr, B.idx, B.v32, B.v64, off,
                                                  ncols, k0, p0);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(tmp2, sort_tmp, k0, k1, p0, p1, (int)nf, 0, bits, st);
    if (e == cudaSuccess) {
        sum_runs<<<grid_for(nf), 256, 0, st>>>(nf, k1, p1, accs, kept);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp2, sum_tmp, kept, pos, (int)nf, st);
    int last_pos = 0, last_kept = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&last_pos, pos + nf - 1, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&last_kept, kept + nf - 1, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    const long long nout = (long long)last_pos + last_kept;
    // compacted (key, value) pairs: reuse k0 / p0
    if (e == cudaSuccess && nout > 0) {
        emit_kept<<<grid_for(nf), 256, 0, st>>>(nf, k1, accs, kept, pos, ncols, k0, p0);
        e = cudaGetLastError();
    }
    cudaFreeAsync(m1, st);
    if (e != cudaSuccess) {
        cudaFreeAsync(m2, st);
        return e;
    }
    out->nnz = nout;
    out->keys_buf = k0;  // (owned by out->mem)
    out->vals_buf = p0;
    out->mem = m2;
    return cudaSuccess;
}

cudaError_t spgemm_finish(const SpgemmOut& o, long long nrows, long long ncols, int32_t* ptr, int32_t* idx, float* v32,
                          double* v64, int* max_len, cudaStream_t st) {
    int* dmax = nullptr;
    cudaError_t e = cudaMallocAsync(&dmax, 4, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(dmax, 0, 4, st);
    if (o.nnz == 0) {
        zero_ptr<<<grid_for(nrows + 1), 256, 0, st>>>(ptr, nrows + 1);
    } else {
        fill_from_keys<<<grid_for(o.nnz), 256, 0, st>>>(o.nnz, o.keys_buf, o.vals_buf, ncols, nrows, ptr, idx, v32,
                                                        v64, dmax);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(max_len, dmax, 4, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(dmax, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e;
}

cudaError_t spgemm_inexact(const SpgemmOut& o, bool* inexact, cudaStream_t st) {
    *inexact = false;
    if (o.nnz == 0) return cudaSuccess;
    int* flag = nullptr;
    cudaError_t e = cudaMallocAsync(&flag, 4, st);
    if (e != cudaSuccess) return e;
    int h = 0;
    e = cudaMemsetAsync(flag, 0, 4, st);
    if (e == cudaSuccess) {
        any_inexact<<<grid_for(o.nnz), 256, 0, st>>>(o.nnz, o.vals_buf, flag);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(flag, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    *inexact = h != 0;
    return e;
}

// P (inc/conv.hpp:125-135): row u*(n+2p)+v holds 1.0 at column (u-p)*n+(v-p)
// when the padded pixel (u, v) is an input pixel.
__global__ void padding_matrix(int m, int n, int p, long long rows, int32_t* ptr, int32_t* idx, float* val) {
    const int w = n + 2 * p;
    for (long long R = blockIdx.x * (long long)blockDim.x + threadIdx.x; R <= rows; R += (long long)gridDim.x * blockDim.x) {
        if (R == rows) {
            ptr[R] = m * n;
            continue;
        }
        const int u = (int)(R / w), v = (int)(R - (long long)u * w);
        const int full = min(max(u - p, 0), m);  // input rows entirely before row u
        const bool urow = u >= p && u < p + m;
        const int before = full * n + (urow ? min(max(v - p, 0), n) : 0);
        ptr[R] = before;
        if (urow && v >= p && v < p + n) {
            idx[before] = (u - p) * n + (v - p);
            val[before] = 1.0f;
        }
    }
}

// C (inc/conv.hpp:141-162): row x*n_out+y holds all k*k taps (zeros included)
// at padded columns (s*x+j)*(n+2p) + s*y+i.
__global__ void conv_matrix(int k, int s, int p, int n, int no, long long rows, const float* t32, const double* t64,
                            int32_t* ptr, int32_t* idx, float* v32, double* v64) {
    const int w = n + 2 * p, kk = k * k;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r <= rows; r += (long long)gridDim.x * blockDim.x) {
        ptr[r] = (int32_t)(r * kk);
        if (r == rows) continue;
        const int x = (int)(r / no), y = (int)(r - (long long)x * no);
        long long e = r * kk;
        for (int j = 0; j < k; ++j)
            for (int i = 0; i < k; ++i, ++e) {
                idx[e] = (s * x + j) * w + s * y + i;
                v32[e] = t32[j * k + i];
                if (v64) v64[e] = t64[j * k + i];
            }
    }
}

cudaError_t launch_padding_matrix(int m, int n, int p, long long rows, int32_t* ptr, int32_t* idx, float* val,
                                  cudaStream_t st) {
    padding_matrix<<<grid_for(rows + 1), 256, 0, st>>>(m, n, p, rows, ptr, idx, val);
    return cudaGetLastError();
}

cudaError_t launch_conv_matrix(int k, int s, int p, int n, int no, long long rows, const float* t32,
                               const double* t64, int32_t* ptr, int32_t* idx, float* v32, double* v64,
                               cudaStream_t st) {
    conv_matrix<<<grid_for(rows + 1), 256, 0, st>>>(k, s, p, n, no, rows, t32, t64, ptr, idx, v32, v64);
    return cudaGetLastError();
}

}  // namespace spb
