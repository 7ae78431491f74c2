// csc_apply.cu -- SpMV / SpMM of a conv transform held in CSC storage, reading
// the CSC storage itself (no row-major copy).
//
// Replaces detail::spmv_csc_cols and spmv's CSC branch (inc/sparse.hpp:194-205,
// 214-258).  The reference scatters column by column:
//     y = 0; for j (column, ascending): for k in ptr[j]..ptr[j+1]: y[idx[k]] += val[k] * x[j]
// so every output sees its entries in ascending column order -- the CSR row
// loop's order.  With nt > 1 reference threads the columns are cut into
// contiguous chunks of ceil(cols / nt); each thread scatters its chunk into a
// partial vector starting from 0.0 and the partials are added to y in thread
// order (inc/sparse.hpp:243-258).
//
// csc_gather<T, KC> -- one thread per output row r = (x, y), any k, s, p, dense
// or zero-tap kernels (the batches of the band geometries go through
// conv_band_check<csc> + conv_spmm_band instead, spmm_band.cu).  The entries of
// row r sit at closed-form places in the CSC storage: tap (j, i) of r lives in
// column (a, b) = (s x + j - p, s y + i - p) at rank
//     #{stored (j', i') of that column with j' > j, or j' == j and i' > i}
// (rows ascend there as j, i descend), i.e. pos = col_ptr[col] + rank.  So the
// thread reads col_ptr[col], then row_idx[pos] and vals[pos] -- every entry of
// the storage is read exactly once per call -- and checks them against (r, the
// tap); the same threads also sweep col_ptr against its closed form
// (csc_build.cu).  Storage equal to the transform of the handle's taps passes
// every comparison; anything else sets the handle's failure flag.  The sums
// themselves run over the stored taps in (j, i) = column-ascending order with
// x gathered per image:
//     fp32: acc = fmaf(w, x, acc)                          (the device contract)
//     fp64: part = part + w * x, two roundings; y = y + part at every chunk
//           boundary -- the reference's fp64 arithmetic and thread order.
#include <algorithm>

#include "internal.h"

namespace spb {

namespace {

// #{x in [0, mo) : 0 <= s x + j - p < a}
__device__ __forceinline__ int slides_below_g(int j, int a, int mo, int s, int p) {
    if (a <= 0) return 0;
    const int lo = p - j <= 0 ? 0 : (p - j + s - 1) / s;
    const int b = a - 1 + p - j;
    if (b < 0) return 0;
    const int hi = min(mo - 1, b / s);
    return max(0, hi - lo + 1);
}

__device__ __forceinline__ void tap_range_g(int x, int dim, int k, int s, int p, int& lo, int& hi) {
    lo = max(0, p - s * x);
    hi = min(k, dim + p - s * x);
    lo = min(lo, k);
    if (hi < lo) hi = lo;
}

template <typename T>
struct Arith;
template <>
struct Arith<float> {
    __device__ static float load(const void* X, long long i) { return __ldg(reinterpret_cast<const float*>(X) + i); }
    __device__ static float step(float acc, float w, float x) { return fmaf(w, x, acc); }
};
template <>
struct Arith<double> {
    __device__ static double load(const void* X, long long i) {
        return __ldg(reinterpret_cast<const double*>(X) + i);
    }
    __device__ static double step(double acc, double w, double x) { return __dadd_rn(acc, __dmul_rn(w, x)); }
};

constexpr int kBT = 4;  // images per pass over a row's taps

}  // namespace

// KC: compile-time kernel side (0: runtime P.k <= 32).
template <typename T, int KC>
__global__ void __launch_bounds__(256) csc_gather(const CscGatherParams P) {
    constexpr bool F64 = sizeof(T) == 8;
    __shared__ T s_w[1024];
    __shared__ uint32_t s_w32[1024];
    const int k = KC ? KC : P.k, kk = k * k, S = P.s;
    for (int q = threadIdx.x; q < kk; q += blockDim.x) {
        const float t32 = __ldg(P.taps32 + q);
        s_w32[q] = __float_as_uint(t32);
        if (F64)
            s_w[q] = (T)(P.taps64 ? __ldg(P.taps64 + q) : (double)t32);
        else
            s_w[q] = (T)t32;
    }
    __syncthreads();
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthr = (long long)gridDim.x * blockDim.x;
    bool bad = false;

    // ---- col_ptr against its closed form (csc_build.cu) ----
    {
        for (long long c = gtid; c <= P.cols; c += nthr) {
            long long want = P.nnz;
            if (c < P.cols) {
                const int a = (int)(c / P.n), b = (int)(c - (long long)a * P.n);
                want = 0;
                uint32_t nzj[KC ? KC : 32];
#pragma unroll
                for (int i = 0; i < (KC ? KC : 32); ++i) nzj[i] = 0;
                for (int j = 0; j < k; ++j) {
                    want += P.zw[j] * slides_below_g(j, a, P.mo, S, P.p);
                    const int d = a + P.p - j;
                    if (d >= 0 && d % S == 0 && d / S < P.mo)
                        for (int i = 0; i < k; ++i) nzj[i] += (P.nzrow[j] >> i) & 1u;
                }
                for (int i = 0; i < k; ++i) want += (long long)nzj[i] * slides_below_g(i, b, P.no, S, P.p);
            }
            bad |= (long long)__ldg(P.col_ptr + c) != want;
        }
    }

    // ---- rows ----
    for (long long r = gtid; r < P.rows; r += nthr) {
        const int x = (int)(r / P.no), y = (int)(r - (long long)x * P.no);
        int jlo, jhi, ilo, ihi;
        tap_range_g(x, P.m, k, S, P.p, jlo, jhi);
        tap_range_g(y, P.n, k, S, P.p, ilo, ihi);
        const long long rb = (long long)(S * x - P.p) * P.n + (S * y - P.p);  // column of tap (0, 0)
        // verification: every stored tap of r at its closed-form place
        for (int j = jlo; j < jhi; ++j) {
            const int idxJ = min((k - 1 - j) / S, x);
            const uint32_t nzr = P.nzrow[j];
            for (int i = ilo; i < ihi; ++i) {
                if (!((nzr >> i) & 1u)) continue;
                const long long col = rb + (long long)j * P.n + i;
                const int idxI = min((k - 1 - i) / S, y);
                int rank;
                if (!P.zt) {
                    const int nI = idxI + 1 + min(i / S, P.no - 1 - y);
                    rank = idxJ * nI + idxI;
                } else {
                    // I(b): taps i' = i + d s with y - d in [0, no)
                    uint32_t mi = 0;
                    for (int d = -min(i / S, P.no - 1 - y); d <= idxI; ++d) mi |= 1u << (i + d * S);
                    rank = __popc(nzr & mi & ~((2u << i) - 1u));
                    for (int d = 1; d <= idxJ; ++d) rank += __popc(P.nzrow[j + d * S] & mi);
                }
                const long long pos = (long long)__ldg(P.col_ptr + col) + rank;
                if (pos < 0 || pos >= P.nnz) {
                    bad = true;
                    continue;
                }
                bad |= __ldg(P.row_idx + pos) != (int)r;
                if (F64 && P.vals64)
                    bad |= __double_as_longlong(__ldg(P.vals64 + pos)) !=
                           __double_as_longlong((double)s_w[j * k + i]);
                else
                    bad |= __float_as_uint(__ldg(P.vals + pos)) != s_w32[j * k + i];
            }
        }
        if (P.verify_only) continue;
        // sums: stored taps in column-ascending order
        for (int b0 = 0; b0 < P.batch; b0 += kBT) {
            T acc[kBT], part[kBT];
#pragma unroll
            for (int u = 0; u < kBT; ++u) acc[u] = part[u] = (T)0;
            long long cur = -1;
            for (int j = jlo; j < jhi; ++j) {
                const uint32_t nzr = P.nzrow[j];
                for (int i = ilo; i < ihi; ++i) {
                    if (!((nzr >> i) & 1u)) continue;
                    const long long col = rb + (long long)j * P.n + i;
                    const T w = s_w[j * k + i];
                    if (F64 && P.chunk > 0) {
                        const long long cid = col / P.chunk;
                        if (cid != cur) {
#pragma unroll
                            for (int u = 0; u < kBT; ++u) {
                                acc[u] = Arith<T>::step(acc[u], (T)1, part[u]);  // y + part (1 * part is exact)
                                part[u] = (T)0;
                            }
                            cur = cid;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kBT; ++u)
                        if (b0 + u < P.batch)
                            part[u] = Arith<T>::step(part[u], w, Arith<T>::load(P.X, (long long)(b0 + u) * P.ldx + col));
                }
            }
#pragma unroll
            for (int u = 0; u < kBT; ++u) {
                if (b0 + u >= P.batch) break;
                const T v = (F64 && P.chunk > 0) ? Arith<T>::step(acc[u], (T)1, part[u]) : part[u];
                reinterpret_cast<T*>(P.Y)[(long long)(b0 + u) * P.ldy + r] = v;
            }
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) *P.fail = 1;
}

// One or two images, k <= 7, dense or zero-tap fp32 taps (the DenseNet
// CSC-SpMV column): the same reads and checks as csc_gather with a row's loads
// issued all at once -- col_ptr of its k^2 columns, then their (row, value)
// entries, both before griddepcontrol.wait (the matrix is never the previous
// kernel's output), then the x gathers -- and the taps in the kernel
// parameters.  Launched as a programmatic dependent, a chained call fetches
// and checks its matrix while the previous kernel runs.
template <int KC>
__global__ void __launch_bounds__(128) csc_gather_lat(const CscGatherParams P) {
    constexpr int KK = KC * KC;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthr = (long long)gridDim.x * blockDim.x;
    const int S = P.s;
    bool bad = false;
    for (long long c = gtid; c <= P.cols; c += nthr) {  // col_ptr against its closed form
        long long want = P.nnz;
        if (c < P.cols) {
            const int a = (int)(c / P.n), b = (int)(c - (long long)a * P.n);
            want = 0;
            int nzj[KC];
#pragma unroll
            for (int i = 0; i < KC; ++i) nzj[i] = 0;
#pragma unroll
            for (int j = 0; j < KC; ++j) {
                want += P.zw[j] * slides_below_g(j, a, P.mo, S, P.p);
                const int d = a + P.p - j;
                if (d >= 0 && d % S == 0 && d / S < P.mo)
#pragma unroll
                    for (int i = 0; i < KC; ++i) nzj[i] += (P.nzrow[j] >> i) & 1u;
            }
#pragma unroll
            for (int i = 0; i < KC; ++i) want += (long long)nzj[i] * slides_below_g(i, b, P.no, S, P.p);
        }
        bad |= (long long)__ldg(P.col_ptr + c) != want;
    }
    const long long r = gtid;
    bool live = r < P.rows;
    int x = 0, y = 0, jlo = 0, jhi = 0, ilo = 0, ihi = 0;
    long long rb = 0;
    if (live) {
        x = (int)(r / P.no);
        y = (int)(r - (long long)x * P.no);
        tap_range_g(x, P.m, KC, S, P.p, jlo, jhi);
        tap_range_g(y, P.n, KC, S, P.p, ilo, ihi);
        rb = (long long)(S * x - P.p) * P.n + (S * y - P.p);
    }
    bool st[KK];
    int cp[KK];
#pragma unroll
    for (int q = 0; q < KK; ++q) {
        const int j = q / KC, i = q - j * KC;
        st[q] = live && j >= jlo && j < jhi && i >= ilo && i < ihi && ((P.nzrow[j] >> i) & 1u);
        cp[q] = st[q] ? __ldg(P.col_ptr + rb + (long long)j * P.n + i) : 0;
    }
    int rw[KK];
    uint32_t vw[KK];
#pragma unroll
    for (int q = 0; q < KK; ++q) {
        const int j = q / KC, i = q - j * KC;
        rw[q] = (int)r;
        vw[q] = __float_as_uint(P.it32[q]);
        if (!st[q]) continue;
        const int idxJ = min((KC - 1 - j) / S, x), idxI = min((KC - 1 - i) / S, y);
        int rank;
        if (!P.zt) {
            rank = idxJ * (idxI + 1 + min(i / S, P.no - 1 - y)) + idxI;
        } else {
            uint32_t mi = 0;
            for (int d = -min(i / S, P.no - 1 - y); d <= idxI; ++d) mi |= 1u << (i + d * S);
            rank = __popc(P.nzrow[j] & mi & ~((2u << i) - 1u));
            for (int d = 1; d <= idxJ; ++d) rank += __popc(P.nzrow[j + d * S] & mi);
        }
        const long long pos = (long long)cp[q] + rank;
        if (pos < 0 || pos >= P.nnz) {
            bad = true;
            continue;
        }
        rw[q] = __ldg(P.row_idx + pos);
        vw[q] = __float_as_uint(__ldg(P.vals + pos));
    }
#pragma unroll
    for (int q = 0; q < KK; ++q)
        if (st[q]) bad |= rw[q] != (int)r || vw[q] != __float_as_uint(P.it32[q]);
    // x may be the previous kernel's output: the gathers wait for it
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (live) {
        for (int b = 0; b < P.batch; ++b) {
            const float* X = reinterpret_cast<const float*>(P.X) + (long long)b * P.ldx;
            float xv[KK];
#pragma unroll
            for (int q = 0; q < KK; ++q) {
                const int j = q / KC, i = q - j * KC;
                xv[q] = st[q] ? __ldg(X + rb + (long long)j * P.n + i) : 0.0f;
            }
            float acc = 0.0f;
#pragma unroll
            for (int q = 0; q < KK; ++q)
                if (st[q]) acc = fmaf(P.it32[q], xv[q], acc);
            reinterpret_cast<float*>(P.Y)[(long long)b * P.ldy + r] = acc;
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) *P.fail = 1;
}

// k >= 5 (25-49 taps a row): four lanes per row.  Lane q of the quad reads and
// checks taps q, q + 4, ... (col_ptr, then the entry, then x), so a row's
// loads are spread over four threads; the quad's first lane then runs the sum
// in (j, i) order, taking each x from the lane that loaded it.
template <int KC>
__global__ void __launch_bounds__(128) csc_gather_lat4(const CscGatherParams P) {
    constexpr int KK = KC * KC, NU = (KK + 3) / 4;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthr = (long long)gridDim.x * blockDim.x;
    const int S = P.s;
    bool bad = false;
    for (long long c = gtid; c <= P.cols; c += nthr) {  // col_ptr against its closed form
        long long want = P.nnz;
        if (c < P.cols) {
            const int a = (int)(c / P.n), b = (int)(c - (long long)a * P.n);
            want = 0;
            int nzj[KC];
#pragma unroll
            for (int i = 0; i < KC; ++i) nzj[i] = 0;
#pragma unroll
            for (int j = 0; j < KC; ++j) {
                want += P.zw[j] * slides_below_g(j, a, P.mo, S, P.p);
                const int d = a + P.p - j;
                if (d >= 0 && d % S == 0 && d / S < P.mo)
#pragma unroll
                    for (int i = 0; i < KC; ++i) nzj[i] += (P.nzrow[j] >> i) & 1u;
            }
#pragma unroll
            for (int i = 0; i < KC; ++i) want += (long long)nzj[i] * slides_below_g(i, b, P.no, S, P.p);
        }
        bad |= (long long)__ldg(P.col_ptr + c) != want;
    }
    const int sub = threadIdx.x & 3, base = (threadIdx.x & 31) & ~3;
    const long long r = gtid >> 2;
    const bool live = r < P.rows;
    int x = 0, y = 0, jlo = 0, jhi = 0, ilo = 0, ihi = 0;
    long long rb = 0;
    if (live) {
        x = (int)(r / P.no);
        y = (int)(r - (long long)x * P.no);
        tap_range_g(x, P.m, KC, S, P.p, jlo, jhi);
        tap_range_g(y, P.n, KC, S, P.p, ilo, ihi);
        rb = (long long)(S * x - P.p) * P.n + (S * y - P.p);
    }
    auto stored = [&](int q) {
        const int j = q / KC, i = q - j * KC;
        return live && q < KK && j >= jlo && j < jhi && i >= ilo && i < ihi && ((P.nzrow[j] >> i) & 1u);
    };
    bool st[NU];
    int cp[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        const int q = sub + 4 * u, j = q / KC, i = q - j * KC;
        st[u] = stored(q);
        cp[u] = st[u] ? __ldg(P.col_ptr + rb + (long long)j * P.n + i) : 0;
    }
    // this lane's taps (compile-time parameter indices, selected by lane)
    uint32_t tw[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        const float t0 = P.it32[4 * u];
        const float t1 = 4 * u + 1 < KK ? P.it32[4 * u + 1] : 0.0f;
        const float t2 = 4 * u + 2 < KK ? P.it32[4 * u + 2] : 0.0f;
        const float t3 = 4 * u + 3 < KK ? P.it32[4 * u + 3] : 0.0f;
        tw[u] = __float_as_uint(sub == 0 ? t0 : sub == 1 ? t1 : sub == 2 ? t2 : t3);
    }
    int rw[NU];
    uint32_t vw[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        const int q = sub + 4 * u, j = q / KC, i = q - j * KC;
        rw[u] = (int)r;
        vw[u] = tw[u];
        if (!st[u]) continue;
        const int idxJ = min((KC - 1 - j) / S, x), idxI = min((KC - 1 - i) / S, y);
        int rank;
        if (!P.zt) {
            rank = idxJ * (idxI + 1 + min(i / S, P.no - 1 - y)) + idxI;
        } else {
            uint32_t mi = 0;
            for (int d = -min(i / S, P.no - 1 - y); d <= idxI; ++d) mi |= 1u << (i + d * S);
            rank = __popc(P.nzrow[j] & mi & ~((2u << i) - 1u));
            for (int d = 1; d <= idxJ; ++d) rank += __popc(P.nzrow[j + d * S] & mi);
        }
        const long long pos = (long long)cp[u] + rank;
        if (pos < 0 || pos >= P.nnz) {
            bad = true;
            continue;
        }
        rw[u] = __ldg(P.row_idx + pos);
        vw[u] = __float_as_uint(__ldg(P.vals + pos));
    }
#pragma unroll
    for (int u = 0; u < NU; ++u)
        if (st[u]) bad |= rw[u] != (int)r || vw[u] != tw[u];
    // x may be the previous kernel's output: the gathers wait for it
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int b = 0; b < P.batch; ++b) {
        const float* X = reinterpret_cast<const float*>(P.X) + (long long)b * P.ldx;
        float xv[NU];
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            const int q = sub + 4 * u, j = q / KC, i = q - j * KC;
            xv[u] = st[u] ? __ldg(X + rb + (long long)j * P.n + i) : 0.0f;
        }
        float acc = 0.0f;
#pragma unroll
        for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float xx = __shfl_sync(0xffffffffu, xv[u], base + t);
                const int q = 4 * u + t;
                if (q < KK && stored(q)) acc = fmaf(P.it32[q], xx, acc);
            }
        if (live && sub == 0) reinterpret_cast<float*>(P.Y)[(long long)b * P.ldy + r] = acc;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) *P.fail = 1;
}

cudaError_t launch_csc_gather_lat(const CscGatherParams& cp, cudaStream_t st, int sms, bool pdl) {
    (void)sms;
    if (cp.batch > 2 || cp.k > 7 || !cp.inline_taps) return cudaErrorInvalidValue;
    const bool quad = cp.k >= 5;
    const long long work = std::max<long long>((quad ? 4 : 1) * cp.rows, cp.cols + 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(((quad ? 4 : 1) * cp.rows + 127) / 128 > 0 ? ((quad ? 4 : 1) * cp.rows + 127) / 128 : 1));
    // (the col_ptr sweep strides over the same threads: enough of them for cols + 1)
    if ((long long)cfg.gridDim.x * 128 < work) cfg.gridDim.x = (unsigned)((work + 127) / 128);
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    switch (cp.k) {
        case 1: return cudaLaunchKernelEx(&cfg, csc_gather_lat<1>, cp);
        case 2: return cudaLaunchKernelEx(&cfg, csc_gather_lat<2>, cp);
        case 3: return cudaLaunchKernelEx(&cfg, csc_gather_lat<3>, cp);
        case 4: return cudaLaunchKernelEx(&cfg, csc_gather_lat<4>, cp);
        case 5: return cudaLaunchKernelEx(&cfg, csc_gather_lat4<5>, cp);
        case 6: return cudaLaunchKernelEx(&cfg, csc_gather_lat4<6>, cp);
        case 7: return cudaLaunchKernelEx(&cfg, csc_gather_lat4<7>, cp);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_csc_gather(const CscGatherParams& cp, bool f64, cudaStream_t st, int sms) {
    if (cp.k > 32) return cudaErrorInvalidValue;
    const long long work = std::max<long long>(cp.rows, cp.cols + 1);
    const long long grid = std::max<long long>(1, std::min<long long>((work + 255) / 256, (long long)sms * 8));
    auto pick = [&](auto kern3, auto kern5, auto kern7, auto kern0) {
        switch (cp.k) {
            case 3: return kern3;
            case 5: return kern5;
            case 7: return kern7;
            default: return kern0;
        }
    };
    if (f64)
        pick(csc_gather<double, 3>, csc_gather<double, 5>, csc_gather<double, 7>, csc_gather<double, 0>)
            <<<(unsigned)grid, 256, 0, st>>>(cp);
    else
        pick(csc_gather<float, 3>, csc_gather<float, 5>, csc_gather<float, 7>, csc_gather<float, 0>)
            <<<(unsigned)grid, 256, 0, st>>>(cp);
    return cudaGetLastError();
}

}  // namespace spb
