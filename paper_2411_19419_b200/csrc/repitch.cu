// repitch.cu -- images whose rows are not 16-byte pitched (odd widths:
// BASELINE config 5's 257 x 193) copied into 16-byte pitched rows, so the
// band apply's windows can be TMA boxes instead of element copies issued by
// one producer warp (spmm_band.cuh load_window).  Reads and writes coalesced
// along each image; the padding columns are never read (the tensor map's row
// length stays n: columns >= n are out of bounds, zero-filled).
#include "internal.h"

namespace spb {

namespace {

constexpr int kThreads = 256, kU = 4;  // elements per thread, loads issued together

// Image blockIdx.y, its elements i = blockIdx.x * (kThreads * kU) + u * kThreads + tid:
// reads and writes coalesced along the flat image, the row split per element.
template <typename T>
__global__ void __launch_bounds__(kThreads) repitch_rows(const T* __restrict__ X, long long ldx, T* __restrict__ Xp,
                                                        int m, int n, long long np) {
    const unsigned total = (unsigned)m * (unsigned)n;
    const T* src = X + (long long)blockIdx.y * ldx;
    T* dst = Xp + (long long)blockIdx.y * m * np;
    const unsigned i0 = blockIdx.x * (kThreads * kU) + threadIdx.x;
    T v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        const unsigned i = i0 + u * kThreads;
        v[u] = i < total ? __ldcs(src + i) : T(0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        const unsigned i = i0 + u * kThreads;
        if (i < total) {
            const unsigned r = i / (unsigned)n;
            dst[(long long)r * np + (i - r * (unsigned)n)] = v[u];
        }
    }
}

}  // namespace

cudaError_t launch_repitch(const void* X, int64_t ldx, void* Xp, int m, int n, int64_t np, int64_t batch, bool f64,
                           cudaStream_t st) {
    const long long total = (long long)m * n;
    if (batch <= 0 || total <= 0) return cudaSuccess;
    if (total > 0xffffffffll - kThreads * kU || batch > 65535) return cudaErrorInvalidValue;
    const dim3 grid((unsigned)((total + kThreads * kU - 1) / (kThreads * kU)), (unsigned)batch);
    if (f64)
        repitch_rows<double><<<grid, kThreads, 0, st>>>(static_cast<const double*>(X), ldx,
                                                         static_cast<double*>(Xp), m, n, np);
    else
        repitch_rows<float><<<grid, kThreads, 0, st>>>(static_cast<const float*>(X), ldx,
                                                        static_cast<float*>(Xp), m, n, np);
    return cudaGetLastError();
}

}  // namespace spb
