// group.cu -- one launch applies a list of CSR transforms, each to its own
// vector (spconv_spmv_group / spconv_convolve_host_group).
//
// The DenseNet121 table (inc/bench.hpp:202-349) is 123 small transforms
// (7^2 .. 224^2 outputs, 1-49 entries a row): applied one kernel at a time,
// the device time is launch-bound (123 launches, ~1 us of work each) and a
// host-buffer call per layer pays the box's ~9 us launch+sync round trip
// (scripts/probe_host_lat.cu).  Here every layer's rows become CTAs of ONE
// grid: CTA b finds its member by a binary search over the members' first
// block, each thread owns one output row and evaluates it exactly as the
// per-layer kernels do -- acc = +0.0f; for e in row (stored order):
// acc = fmaf(vals[e], x[col_idx[e]], acc) -- so the outputs are bit-identical
// to spconv_spmv on each member (the reference's row loop,
// inc/sparse.hpp:180-192, evaluated in fp32 with fmaf).  The fp64 form
// evaluates the reference's own arithmetic -- acc = acc + val * x, one rounded
// multiply and one rounded add per entry -- and is bit-identical to the
// reference's spmv() (and to spconv_spmm_f64) on each member.
//
// Loads are issued in groups of G entries (all column indices and values,
// then all x gathers), so a 9-entry row costs three dependent round trips
// (row_ptr, entries, x) whatever its length up to G.
#include <type_traits>

#include "internal.h"

namespace spb {

namespace {

constexpr int kThreads = 128;
constexpr int kG = 16;
constexpr int kQ = 13;  // entries per lane and pass in the four-lanes-per-row form (52 a row)

template <bool F64>
__global__ void __launch_bounds__(kThreads) csr_spmv_group(const GroupParams P) {
    using T = typename std::conditional<F64, double, float>::type;
    // member owning this block: the last m with blk0[m] <= blockIdx.x
    int lo = 0, hi = P.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (P.m[mid].blk0 <= (int)blockIdx.x) lo = mid;
        else hi = mid - 1;
    }
    const GroupMember& M = P.m[lo];
    const T* x = static_cast<const T*>(M.x);
    if (M.quad) {
        // Rows longer than 16 entries (k = 5, 7 layers): four lanes per row
        // load the row's entries together (lane q of the quad: entries q, q + 4,
        // ...), so a 49-entry row costs the same three round trips as a short
        // one; the quad's first lane then runs the ordered chain, taking each
        // (value, x) pair from the lane that loaded it.
        const int sub = threadIdx.x & 3, base = (threadIdx.x & 31) & ~3;
        const int r = (((int)blockIdx.x - M.blk0) * kThreads + (int)threadIdx.x) >> 2;
        const bool live = r < M.rows;
        const int e0 = live ? __ldg(M.row_ptr + r) : 0, e1 = live ? __ldg(M.row_ptr + r + 1) : 0;
        T acc = 0;
        // (warp-uniform trip count: the shuffles need every lane)
        const int nmax = __reduce_max_sync(0xffffffffu, e1 - e0);
        for (int o = 0; o < nmax; o += 4 * kQ) {
            const int e = e0 + o;
            int c[kQ];
            T v[kQ], xv[kQ];
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                const int ee = e + sub + 4 * q;
                c[q] = ee < e1 ? __ldg(M.col_idx + ee) : 0;
                if constexpr (F64)
                    v[q] = ee < e1 ? (M.vals64 ? __ldg(M.vals64 + ee) : (double)__ldg(M.vals + ee)) : 0.0;
                else
                    v[q] = ee < e1 ? __ldg(M.vals + ee) : 0.0f;
            }
#pragma unroll
            for (int q = 0; q < kQ; ++q) xv[q] = e + sub + 4 * q < e1 ? __ldg(x + c[q]) : T(0);
#pragma unroll
            for (int q = 0; q < kQ; ++q)
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const T vv = __shfl_sync(0xffffffffu, v[q], base + t);
                    const T xx = __shfl_sync(0xffffffffu, xv[q], base + t);
                    if (e + 4 * q + t < e1) {
                        if constexpr (F64)
                            acc = __dadd_rn(acc, __dmul_rn(vv, xx));
                        else
                            acc = fmaf(vv, xx, acc);
                    }
                }
        }
        if (live && sub == 0) static_cast<T*>(M.y)[r] = acc;
        return;
    }
    const int r = ((int)blockIdx.x - M.blk0) * kThreads + (int)threadIdx.x;
    if (r >= M.rows) return;
    const int e0 = __ldg(M.row_ptr + r), e1 = __ldg(M.row_ptr + r + 1);
    T acc = 0;
    for (int e = e0; e < e1; e += kG) {
        int c[kG];
        T v[kG], xv[kG];
#pragma unroll
        for (int q = 0; q < kG; ++q) {
            c[q] = e + q < e1 ? __ldg(M.col_idx + e + q) : 0;
            if constexpr (F64)
                v[q] = e + q < e1 ? (M.vals64 ? __ldg(M.vals64 + e + q) : (double)__ldg(M.vals + e + q)) : 0.0;
            else
                v[q] = e + q < e1 ? __ldg(M.vals + e + q) : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < kG; ++q) xv[q] = e + q < e1 ? __ldg(x + c[q]) : T(0);
#pragma unroll
        for (int q = 0; q < kG; ++q)
            if (e + q < e1) {
                if constexpr (F64)  // the reference's rounded multiply, then rounded add (inc/sparse.hpp:185-191)
                    acc = __dadd_rn(acc, __dmul_rn(v[q], xv[q]));
                else
                    acc = fmaf(v[q], xv[q], acc);
            }
    }
    static_cast<T*>(M.y)[r] = acc;
}

}  // namespace

cudaError_t launch_spmv_group(const GroupParams& gp, int blocks, bool f64, cudaStream_t st) {
    if (gp.count <= 0 || blocks <= 0) return cudaSuccess;
    if (f64)
        csr_spmv_group<true><<<blocks, kThreads, 0, st>>>(gp);
    else
        csr_spmv_group<false><<<blocks, kThreads, 0, st>>>(gp);
    return cudaGetLastError();
}

int group_blocks(int64_t rows, bool quad) { return (int)(((quad ? 4 : 1) * rows + kThreads - 1) / kThreads); }

}  // namespace spb
