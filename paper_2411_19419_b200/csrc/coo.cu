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
