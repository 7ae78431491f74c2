// csr_build.cu -- one-pass on-device construction of the CSR of T = C*P.
//
// Replaces build_transform (inc/conv.hpp:179-204): build_conv_matrix (:141-162)
// + build_padding_matrix (:125-135) + spgemm (inc/sparse.hpp:296-342) +
// SparseMatrix::compile (inc/sparse.hpp:85-119).  Nothing is sorted and no
// intermediate C or P exists: each row's entries are generated directly in
// their final (column-ascending) order.
//
// Row r = x*n_out + y (inc/conv.hpp:8-12) keeps tap (j,i) iff the tap lands in
// the input, i.e. j in J(x) = [jlo(x), jhi(x)), i in I(y) = [ilo(y), ihi(y)),
//   jlo = max(0, p - s*x),  jhi = min(k, m + p - s*x)        (and likewise i),
// -- the paper's max(0, k - c1(x)) * max(0, k - c2(y)) count
// (inc/analysis.hpp:21-52) -- AND the tap is not an exact zero
// (inc/sparse.hpp:335, inc/conv.hpp:201).  Its column is
//   (s*x + j - p)*n + (s*y + i - p).
// The count is a summed-area-table query over the (tap != 0) mask, which
// reduces to the closed form when no tap is zero.
//
// row_ptr is closed-form as well.  With W[j] = sum_i nz[j][i] * #{y : i in I(y)}
// (host, O(k^2)), the number of entries in all rows before (x0, y0) is
//   sum_j W[j] * #{x' < x0 : j in J(x')}  +  sum_i nzcol(x0, i) * #{y' < y0 : i in I(y')}
// and both counts are O(1) ranges, so every CTA computes its global offset in
// O(k) without a grid-wide scan or look-back; a block scan of the per-row
// counts finishes row_ptr.  Entries are staged in shared memory at the global
// offset's alignment and written back with 16-byte streaming stores, so HBM
// sees each of the 8*nnz + 4*(rows+1) bytes exactly once.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.h"
#include "tma.cuh"

namespace spb {

namespace {

__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ int sat_rect(const int32_t* sat, int k1, int jlo, int jhi, int ilo,
                                        int ihi) {
    return sat[jhi * k1 + ihi] - sat[jlo * k1 + ihi] - sat[jhi * k1 + ilo] + sat[jlo * k1 + ilo];
}

// Valid tap range [lo, hi) along one axis for slide position x (see header).
__device__ __forceinline__ void tap_range(int x, int dim, int k, int s, int p, int& lo, int& hi) {
    lo = max(0, p - s * x);
    hi = min(k, dim + p - s * x);
    lo = min(lo, k);
    if (hi < lo) hi = lo;
}

// #{x' in [0, x) : tap index j in J(x')}  (an O(1) range count).
__device__ __forceinline__ int slides_before(int x, int j, int dim, int s, int p) {
    const int lo = (p - j <= 0) ? 0 : (p - j + s - 1) / s;
    const int hi = (dim + p - j - 1 < 0) ? 0 : (dim + p - j - 1) / s + 1;
    return max(0, min(x, hi) - lo);
}

}  // namespace

// KC = compile-time kernel side (0: runtime P.k).  DENSE: every tap is
// non-zero, so the zero-tap test folds away.
template <int KC, bool DENSE, bool F64 = false>
__global__ void __launch_bounds__(256) csr_build_kernel(const BuildParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_warp[32];
    __shared__ long long s_red[32];

    const int t = threadIdx.x;
    const int R = blockDim.x;
    const int nw = R >> 5;
    const int lane = t & 31, wid = t >> 5;
    const int k = KC ? KC : P.k;
    const int k1 = k + 1, kk = k * k;

    // Tables -> shared memory: sat[(k+1)^2] ints, taps[k^2] floats, then the staging area.
    int32_t* s_sat = reinterpret_cast<int32_t*>(smem);
    float* s_taps = reinterpret_cast<float*>(s_sat + k1 * k1);
    const int tab_words = (k1 * k1 + kk + 3) & ~3;
    for (int q = t; q < k1 * k1; q += R) s_sat[q] = P.small ? P.tab.sat[q] : __ldg(P.t.sat + q);
    for (int q = t; q < kk; q += R) s_taps[q] = P.small ? P.tab.taps[q] : __ldg(P.t.taps + q);
    __syncthreads();
    if (blockIdx.x == 0 && P.taps_out)
        for (int q = t; q < kk; q += R) P.taps_out[q] = s_taps[q];

    const int r0 = blockIdx.x * R;
    const int r = r0 + t;
    const int x0 = r0 / P.no, y0 = r0 - x0 * P.no;  // (block-uniform: one division)

    // ---- per-row count (Theorem 2.1 with the zero-tap mask) ----
    int cnt = 0, x = 0, y = 0, jlo = 0, jhi = 0, ilo = 0, ihi = 0;
    if (r < P.rows) {
        x = x0;
        y = y0 + t;
        if (y >= P.no) {  // the block spans image rows: at most a few wraps unless n_out is tiny
            x += y / P.no;
            y -= (y / P.no) * P.no;
        }
        tap_range(x, P.m, k, P.s, P.p, jlo, jhi);
        tap_range(y, P.n, k, P.s, P.p, ilo, ihi);
        cnt = DENSE ? (jhi - jlo) * (ihi - ilo) : sat_rect(s_sat, k1, jlo, jhi, ilo, ihi);
    }

    // ---- closed-form global offset of row r0 = (x0, y0) ----
    int jlo0, jhi0;
    tap_range(x0, P.m, k, P.s, P.p, jlo0, jhi0);
    long long part = 0;
    for (int q = t; q < k; q += R) {
        const long long wj = P.small ? P.tab.w[q] : __ldg(P.t.w + q);
        part += wj * slides_before(x0, q, P.m, P.s, P.p);
        const int cz = sat_rect(s_sat, k1, jlo0, jhi0, q, q + 1);
        part += (long long)cz * slides_before(y0, q, P.n, P.s, P.p);
    }
    part = warp_sum64(part);
    if (lane == 0) s_red[wid] = part;

    // ---- block exclusive scan of counts ----
    const int inc = warp_incl_scan(cnt);
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int wv = lane < nw ? s_warp[lane] : 0;
        long long pr = lane < nw ? s_red[lane] : 0;
        wv = warp_incl_scan(wv);
        pr = warp_sum64(pr);
        s_warp[lane] = wv;
        if (lane == 0) s_red[0] = pr;
    }
    __syncthreads();
    const int excl = inc - cnt + (wid > 0 ? s_warp[wid - 1] : 0);
    const int total = s_warp[nw - 1];
    const int base = (int)s_red[0];

    if (r < P.rows) {
        P.row_ptr[r] = base + excl;
        if (r == P.rows - 1) P.row_ptr[P.rows] = base + excl + cnt;
    }

    // ---- fill: taps of this row in (j, i) order == column-ascending ----
    const int mis = base & 3;  // stage at the global offset's 16-byte phase
    int32_t* dcol;
    float* dval;
    int o;
    // compile-time for the unrolled k (always staged): shared, not generic, accesses
    const bool staged = KC > 0 || P.stage != 0;
    // F64 (exact-fp64 builds, unrolled k): the fp64 values staged after dval
    double* dv64 = reinterpret_cast<double*>(reinterpret_cast<int32_t*>(smem) + tab_words + 2 * P.stage_words);
    const int mis64 = base & 1;
    int o64 = mis64 + excl;
    if (staged) {
        dcol = reinterpret_cast<int32_t*>(smem) + tab_words;
        dval = reinterpret_cast<float*>(dcol) + P.stage_words;
        o = mis + excl;
    } else {
        dcol = P.col_idx;
        dval = P.vals;
        o = base + excl;
    }
    if (r < P.rows && cnt > 0) {
        const int xr = P.s * x - P.p, yc = P.s * y - P.p;
        if (KC && DENSE && cnt == KC * KC) {
            // Interior row (every tap stored): the K x K pattern, no predicates.
#pragma unroll
            for (int j = 0; j < KC; ++j) {
                const int rowbase = (xr + j) * P.n + yc;
#pragma unroll
                for (int i = 0; i < KC; ++i) {
                    dcol[o + j * KC + i] = rowbase + i;
                    dval[o + j * KC + i] = F64 ? P.f64_t32[j * KC + i] : s_taps[j * KC + i];
                    if (F64) dv64[o64 + j * KC + i] = P.f64_t64[j * KC + i];
                }
            }
        } else if (KC) {
            // Fully unrolled K x K pattern; clipped / zero taps are predicated off.
#pragma unroll
            for (int j = 0; j < KC; ++j) {
                const int rowbase = (xr + j) * P.n + yc;
                const bool jin = j >= jlo && j < jhi;
#pragma unroll
                for (int i = 0; i < KC; ++i) {
                    const float v = s_taps[j * KC + i];
                    const bool keep = jin && i >= ilo && i < ihi && (DENSE || v != 0.0f);
                    if (keep) {
                        dcol[o] = rowbase + i;
                        dval[o] = F64 ? P.f64_t32[j * KC + i] : v;
                        if (F64) dv64[o64] = P.f64_t64[j * KC + i];
                    }
                    o += keep ? 1 : 0;
                    o64 += keep ? 1 : 0;
                }
            }
        } else {
            for (int j = jlo; j < jhi; ++j) {
                const int rowbase = (xr + j) * P.n + yc;
                const float* tj = s_taps + j * k;
                for (int i = ilo; i < ihi; ++i) {
                    const float v = tj[i];
                    if (v != 0.0f) {  // drops +-0.0, keeps NaN (inc/sparse.hpp:335)
                        dcol[o] = rowbase + i;
                        dval[o] = v;
                        ++o;
                    }
                }
            }
        }
    }
    if (staged) {
        if (P.bulk_store) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        // Global [base, base + total) <- staged [mis, mis + total): scalar head,
        // 16-byte body, scalar tail.
        const int head = min(total, (4 - mis) & 3);
        if (t < head) {
            __stcs(P.col_idx + base + t, dcol[mis + t]);
            __stcs(P.vals + base + t, dval[mis + t]);
        }
        const int nvec = (total - head) >> 2;
        const int4* scol = reinterpret_cast<const int4*>(dcol + mis + head);
        const float4* sval = reinterpret_cast<const float4*>(dval + mis + head);
        int4* gcol = reinterpret_cast<int4*>(P.col_idx + base + head);
        float4* gval = reinterpret_cast<float4*>(P.vals + base + head);
        const int head64 = min(total, mis64), nvec64 = (total - head64) >> 1;  // (F64: 2 doubles / 16 B)
        if (F64 && t < head64) __stcs(P.vals64 + base + t, dv64[mis64 + t]);
        if (P.bulk_store) {  // the 16-byte body through the TMA engine: two instructions
            if (t == 0 && (nvec > 0 || (F64 && nvec64 > 0))) {
                if (nvec > 0) {
                    bulk_s2g(gcol, scol, (uint32_t)nvec * 16u);
                    bulk_s2g(gval, sval, (uint32_t)nvec * 16u);
                }
                if (F64 && nvec64 > 0)
                    bulk_s2g(P.vals64 + base + head64, dv64 + mis64 + head64, (uint32_t)nvec64 * 16u);
                bulk_commit_wait_read();
            }
        } else {
            for (int q = t; q < nvec; q += R) {
                __stcs(gcol + q, scol[q]);
                __stcs(gval + q, sval[q]);
            }
            if (F64)
                for (int q = t; q < nvec64; q += R)
                    __stcs(reinterpret_cast<double2*>(P.vals64 + base + head64) + q,
                           reinterpret_cast<const double2*>(dv64 + mis64 + head64)[q]);
        }
        const int done = head + 4 * nvec;
        if (t < total - done) {
            __stcs(P.col_idx + base + done + t, dcol[mis + done + t]);
            __stcs(P.vals + base + done + t, dval[mis + done + t]);
        }
        const int done64 = head64 + 2 * nvec64;
        if (F64 && t < total - done64) __stcs(P.vals64 + base + done64 + t, dv64[mis64 + done64 + t]);
    }
}


// Warp-local variant (the default for the unrolled k): each warp owns 32
// consecutive rows, finds its global offset in closed form (lanes over the k
// tap indices, a warp reduction), scans its counts with shuffles, stages its
// entries in its own shared-memory slice and streams them out with 16-byte
// stores -- no block-wide barrier after the table load, so a warp never waits
// for the slowest warp of its CTA (the block version's dominant stall).
template <int KC, bool DENSE>
__global__ void __launch_bounds__(256) csr_build_warp(const BuildParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int K1 = KC + 1, KK = KC * KC;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    int32_t* s_sat = reinterpret_cast<int32_t*>(smem);
    float* s_taps = reinterpret_cast<float*>(s_sat + K1 * K1);
    constexpr int TAB_WORDS = (K1 * K1 + KK + 3) & ~3;
    for (int q = t; q < K1 * K1; q += blockDim.x) s_sat[q] = P.small ? P.tab.sat[q] : __ldg(P.t.sat + q);
    for (int q = t; q < KK; q += blockDim.x) s_taps[q] = P.small ? P.tab.taps[q] : __ldg(P.t.taps + q);
    __syncthreads();
    if (blockIdx.x == 0 && P.taps_out)
        for (int q = t; q < KK; q += blockDim.x) P.taps_out[q] = s_taps[q];

    const int r0 = (blockIdx.x * (blockDim.x >> 5) + wid) * 32;
    if (r0 >= P.rows) return;
    const int r = r0 + lane;
    int cnt = 0, x = 0, y = 0, jlo = 0, jhi = 0, ilo = 0, ihi = 0;
    if (r < P.rows) {
        x = r / P.no;
        y = r - x * P.no;
        tap_range(x, P.m, KC, P.s, P.p, jlo, jhi);
        tap_range(y, P.n, KC, P.s, P.p, ilo, ihi);
        cnt = DENSE ? (jhi - jlo) * (ihi - ilo) : sat_rect(s_sat, K1, jlo, jhi, ilo, ihi);
    }
    // closed-form global offset of row r0 = (x0, y0)
    const int x0 = r0 / P.no, y0 = r0 - x0 * P.no;
    long long part = 0;
    if (lane < KC) {
        int jlo0, jhi0;
        tap_range(x0, P.m, KC, P.s, P.p, jlo0, jhi0);
        const long long wj = P.small ? P.tab.w[lane] : __ldg(P.t.w + lane);
        part = wj * slides_before(x0, lane, P.m, P.s, P.p) +
               (long long)sat_rect(s_sat, K1, jlo0, jhi0, lane, lane + 1) * slides_before(y0, lane, P.n, P.s, P.p);
    }
    const int base = (int)warp_sum64(part);
    const int inc = warp_incl_scan(cnt);
    const int excl = inc - cnt;
    const int total = __shfl_sync(0xffffffffu, inc, 31);
    if (r < P.rows) {
        P.row_ptr[r] = base + excl;
        if (r == P.rows - 1) P.row_ptr[P.rows] = base + excl + cnt;
    }
    // stage this warp's entries at the global offset's 16-byte phase
    const int mis = base & 3;
    int32_t* dcol = reinterpret_cast<int32_t*>(smem) + TAB_WORDS + wid * 2 * P.stage_words;
    float* dval = reinterpret_cast<float*>(dcol + P.stage_words);
    int o = mis + excl;
    if (r < P.rows && cnt > 0) {
        const int xr = P.s * x - P.p, yc = P.s * y - P.p;
#pragma unroll
        for (int j = 0; j < KC; ++j) {
            const int rowbase = (xr + j) * P.n + yc;
            const bool jin = j >= jlo && j < jhi;
#pragma unroll
            for (int i = 0; i < KC; ++i) {
                const float v = s_taps[j * KC + i];
                const bool keep = jin && i >= ilo && i < ihi && (DENSE || v != 0.0f);
                if (keep) {
                    dcol[o] = rowbase + i;
                    dval[o] = v;
                }
                o += keep ? 1 : 0;
            }
        }
    }
    if (P.bulk_store) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const int head = min(total, (4 - mis) & 3);
    if (lane < head) {
        __stcs(P.col_idx + base + lane, dcol[mis + lane]);
        __stcs(P.vals + base + lane, dval[mis + lane]);
    }
    const int nvec = (total - head) >> 2;
    const int4* scol = reinterpret_cast<const int4*>(dcol + mis + head);
    const float4* sval = reinterpret_cast<const float4*>(dval + mis + head);
    int4* gcol = reinterpret_cast<int4*>(P.col_idx + base + head);
    float4* gval = reinterpret_cast<float4*>(P.vals + base + head);
    if (P.bulk_store) {
        if (lane == 0 && nvec > 0) {
            bulk_s2g(gcol, scol, (uint32_t)nvec * 16u);
            bulk_s2g(gval, sval, (uint32_t)nvec * 16u);
            bulk_commit_wait_read();
        }
    } else {
        for (int q = lane; q < nvec; q += 32) {
            __stcs(gcol + q, scol[q]);
            __stcs(gval + q, sval[q]);
        }
    }
    const int done = head + 4 * nvec;
    if (lane < total - done) {
        __stcs(P.col_idx + base + done + lane, dcol[mis + done + lane]);
        __stcs(P.vals + base + done + lane, dval[mis + done + lane]);
    }
}

// Persistent, double-buffered variant (unrolled k, staged): a grid of a few
// CTAs per SM walks tiles of 256 rows.  Every row's global offset is closed
// form -- sum_j W[j] * #{x' < x : j in J(x')} + sum_i nzcol(x, i) *
// #{y' < y : i in I(y')}, the slide counts from per-tap [lo, hi) tables in
// shared memory -- so there is no scan: a tile costs two CTA barriers, and
// the TMA bulk store of tile t drains while tile t + 1 is generated in the
// other staging buffer.
template <int KC, bool DENSE, bool F64 = false>
__global__ void __launch_bounds__(256) csr_build_persist(const BuildParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int K1 = KC + 1, KK = KC * KC, R = 256;
    constexpr int STAGE = (R * KK + 3 + 3) & ~3;  // words per staging array
    const int t = threadIdx.x;
    __shared__ int32_t s_sat[K1 * K1];
    __shared__ float s_taps[KK];
    __shared__ long long s_w[KC];
    __shared__ int s_xlo[KC], s_xhi[KC], s_ylo[KC], s_yhi[KC];
    for (int q = t; q < K1 * K1; q += R) s_sat[q] = P.small ? P.tab.sat[q] : __ldg(P.t.sat + q);
    for (int q = t; q < KK; q += R) s_taps[q] = P.small ? P.tab.taps[q] : __ldg(P.t.taps + q);
    // F64 (exact-fp64 builds): the taps above are tags; these are their values
    __shared__ float s_r32[F64 ? KK : 1];
    __shared__ double s_r64[F64 ? KK : 1];
    if (F64)
        for (int q = t; q < KK; q += R) {
            s_r32[q] = P.f64_t32[q];
            s_r64[q] = P.f64_t64[q];
        }
    for (int q = t; q < KC; q += R) {
        s_w[q] = P.small ? P.tab.w[q] : __ldg(P.t.w + q);
        // x' with tap q in J(x'): [xlo, xhi) (slides_before(x, q) = clamp(x, xlo, xhi) - xlo)
        s_xlo[q] = (P.p - q <= 0) ? 0 : (P.p - q + P.s - 1) / P.s;
        s_xhi[q] = max(s_xlo[q], (P.m + P.p - q - 1 < 0) ? 0 : (P.m + P.p - q - 1) / P.s + 1);
        s_ylo[q] = (P.p - q <= 0) ? 0 : (P.p - q + P.s - 1) / P.s;
        s_yhi[q] = max(s_ylo[q], (P.n + P.p - q - 1 < 0) ? 0 : (P.n + P.p - q - 1) / P.s + 1);
    }
    __syncthreads();
    if (blockIdx.x == 0 && P.taps_out)
        for (int q = t; q < KK; q += R) P.taps_out[q] = s_taps[q];

    // global offset of row (x, y) and its entry count
    auto row_offset = [&](int x, int y, int& cnt, int& jlo, int& jhi, int& ilo, int& ihi) -> int {
        tap_range(x, P.m, KC, P.s, P.p, jlo, jhi);
        tap_range(y, P.n, KC, P.s, P.p, ilo, ihi);
        cnt = DENSE ? (jhi - jlo) * (ihi - ilo) : sat_rect(s_sat, K1, jlo, jhi, ilo, ihi);
        long long off = 0;
#pragma unroll
        for (int q = 0; q < KC; ++q) {
            const int sx = max(0, min(x, s_xhi[q]) - s_xlo[q]);
            const int sy = max(0, min(y, s_yhi[q]) - s_ylo[q]);
            const int nzc = DENSE ? (jhi - jlo) : sat_rect(s_sat, K1, jlo, jhi, q, q + 1);
            off += s_w[q] * sx + (long long)nzc * sy;
        }
        return (int)off;
    };

    const int ntiles = (P.rows + R - 1) / R;
    __shared__ int s_base[2], s_end[2];
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        // per buffer: col, val (STAGE words each) and, for F64, STAGE doubles
        int32_t* dcol = reinterpret_cast<int32_t*>(smem) + buf * (F64 ? 4 : 2) * STAGE;
        float* dval = reinterpret_cast<float*>(dcol + STAGE);
        double* dv64 = reinterpret_cast<double*>(dcol + 2 * STAGE);
        const int r0 = tile * R;
        const int r1 = min(P.rows, r0 + R);
        // this thread's row: closed-form offset, written to row_ptr now
        const int r = r0 + t;
        int x = 0, y = 0, cnt = 0, off = 0, jlo = 0, jhi = 0, ilo = 0, ihi = 0;
        if (r < r1) {
            x = r / P.no;
            y = r - x * P.no;
            off = row_offset(x, y, cnt, jlo, jhi, ilo, ihi);
            P.row_ptr[r] = off;
            if (r == P.rows - 1) P.row_ptr[P.rows] = off + cnt;
        }
        // the tile's [base, end): row r0's offset and row (r1 - 1)'s end
        if (t == 0) {
            s_base[buf] = off;
            bulk_wait_read<1>();  // this buffer's bulk store of two tiles ago has read it
        }
        if (r == r1 - 1) s_end[buf] = off + cnt;
        __syncthreads();
        const int base = s_base[buf], total = s_end[buf] - base;
        const int mis = base & 3;
        const int mis64 = base & 1;  // (doubles: 16-byte phase)
        if (r < r1) {
            int o = mis + off - base;
            int o64 = mis64 + off - base;
            const int xr = P.s * x - P.p, yc = P.s * y - P.p;
            if (DENSE && cnt == KK) {
#pragma unroll
                for (int j = 0; j < KC; ++j)
#pragma unroll
                    for (int i = 0; i < KC; ++i) {
                        dcol[o + j * KC + i] = (xr + j) * P.n + yc + i;
                        dval[o + j * KC + i] = F64 ? s_r32[j * KC + i] : s_taps[j * KC + i];
                        if (F64) dv64[o64 + j * KC + i] = s_r64[j * KC + i];
                    }
            } else {
#pragma unroll
                for (int j = 0; j < KC; ++j) {
                    const int rowbase = (xr + j) * P.n + yc;
                    const bool jin = j >= jlo && j < jhi;
#pragma unroll
                    for (int i = 0; i < KC; ++i) {
                        const float v = s_taps[j * KC + i];
                        const bool keep = jin && i >= ilo && i < ihi && (DENSE || v != 0.0f);
                        if (keep) {
                            dcol[o] = rowbase + i;
                            dval[o] = F64 ? s_r32[j * KC + i] : v;
                            if (F64) dv64[o64] = s_r64[j * KC + i];
                        }
                        o += keep ? 1 : 0;
                        o64 += keep ? 1 : 0;
                    }
                }
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        const int head = min(total, (4 - mis) & 3);
        if (t < head) {
            __stcs(P.col_idx + base + t, dcol[mis + t]);
            __stcs(P.vals + base + t, dval[mis + t]);
        }
        const int nvec = (total - head) >> 2;
        const int head64 = min(total, mis64), nvec64 = (total - head64) >> 1;  // (F64)
        if (F64 && t < head64) __stcs(P.vals64 + base + t, dv64[mis64 + t]);
        if (t == 0) {
            if (nvec > 0) {
                bulk_s2g(P.col_idx + base + head, dcol + mis + head, (uint32_t)nvec * 16u);
                bulk_s2g(P.vals + base + head, dval + mis + head, (uint32_t)nvec * 16u);
            }
            if (F64 && nvec64 > 0) bulk_s2g(P.vals64 + base + head64, dv64 + mis64 + head64, (uint32_t)nvec64 * 16u);
            bulk_commit();
        }
        const int done = head + 4 * nvec;
        if (t < total - done) {
            __stcs(P.col_idx + base + done + t, dcol[mis + done + t]);
            __stcs(P.vals + base + done + t, dval[mis + done + t]);
        }
        const int done64 = head64 + 2 * nvec64;
        if (F64 && t < total - done64) __stcs(P.vals64 + base + done64 + t, dv64[mis64 + done64 + t]);
    }
    if (t == 0) bulk_wait_read<0>();
}

template <int KC, bool DENSE, bool F64>
static cudaError_t launch_p_f(const BuildParams& bp, cudaStream_t st) {
    constexpr int KK = KC * KC;
    const size_t smem = (size_t)((256 * KK + 3 + 3) & ~3) * 4 * 2 * (F64 ? 4 : 2);  // 2 buffers
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto kern = csr_build_persist<KC, DENSE, F64>;
    static std::atomic<int> occ[64];  // per device, queried once (0 = not yet)
    if (!occ[dev & 63]) {
        int o = 0;
        cudaError_t e = cudaSuccess;
        if (smem > 48 * 1024) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, 256, smem);
        if (e != cudaSuccess) return e;
        occ[dev & 63] = std::max(o, 1);
    }
    const int per_sm = occ[dev & 63];
    const long long tiles = ((long long)bp.rows + 255) / 256;
    const long long grid = std::min<long long>(tiles, (long long)sms * std::max(per_sm, 1));
    kern<<<(unsigned)grid, 256, smem, st>>>(bp);
    return cudaGetLastError();
}

template <int KC, bool DENSE>
static cudaError_t launch_p(const BuildParams& bp, cudaStream_t st) {
    // (F64 instantiations for k <= 5: three staged arrays per buffer)
    if (bp.vals64 && KC <= 5) return launch_p_f<KC, DENSE, KC <= 5>(bp, st);
    return launch_p_f<KC, DENSE, false>(bp, st);
}

template <int KC, bool DENSE>
static cudaError_t launch_w(BuildParams bp, cudaStream_t st) {
    constexpr int KK = KC * KC;
    const size_t tab_bytes = (size_t)(((KC + 1) * (KC + 1) + KK + 3) & ~3) * 4;
    bp.stage_words = (32 * KK + 3 + 3) & ~3;
    const size_t per_warp = (size_t)bp.stage_words * 8;
    int warps = 8;
    while (warps > 1 && tab_bytes + warps * per_warp > 100 * 1024) warps >>= 1;
    const size_t smem = tab_bytes + warps * per_warp;
    static std::atomic<bool> attr[64];  // per device (benign concurrent first use)
    int dev = 0;
    cudaGetDevice(&dev);
    if (smem > 48 * 1024 && !attr[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(csr_build_warp<KC, DENSE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             100 * 1024 + (int)tab_bytes);
        if (e != cudaSuccess) return e;
        attr[dev & 63] = true;
    }
    const long long grid = ((long long)bp.rows + 32 * warps - 1) / (32 * warps);
    csr_build_warp<KC, DENSE><<<(unsigned)grid, 32 * warps, smem, st>>>(bp);
    return cudaGetLastError();
}

template <int KC, bool DENSE>
static cudaError_t launch_k(const BuildParams& bp, int block, size_t smem, cudaStream_t st) {
    // exact-fp64 builds (unrolled k): a third staging array of doubles
    const bool f64 = KC > 0 && bp.vals64 && bp.stage;
    if (f64) smem += (size_t)bp.stage_words * 8;
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    auto kern = f64 ? csr_build_kernel<KC, DENSE, (KC > 0)> : csr_build_kernel<KC, DENSE, false>;
    // the opt-in limit is set once per device to the 200 KB cap every launch
    // respects (a per-launch value could race with another thread's launch)
    static std::atomic<bool> attr[2][64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[f64 ? 1 : 0][dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
        attr[f64 ? 1 : 0][dev & 63] = true;
    }
    const int grid = (bp.rows + block - 1) / block;
    kern<<<grid, block, smem, st>>>(bp);
    return cudaGetLastError();
}

cudaError_t launch_csr_build(const BuildParams& bp_in, bool dense, int block, size_t smem, bool* f64_done,
                             cudaStream_t st) {
    // The exact-fp64 fill exists in the persistent kernel for k <= 5; other
    // launches build the tags only (the caller retags).
    BuildParams bp = bp_in;
    // Default: the persistent double-buffered kernel for k <= 5 (config 3
    // build 22.5 -> 18.4 us, config 2 12.3 -> 10.2 us), the block kernel for
    // larger k, whose 256-row double buffer would not leave room for a second
    // CTA per SM (config 4: block 252 us, persistent 297 us; the block kernel
    // also beats the warp-local one, 254 vs 283 us, profiles/r01_choices).
    // Option build = block | warp | persist forces a kernel.
    const int bsel = opt(kOptBuild);
    const bool warp_build = bsel == 2;
    // (exact-fp64 builds: the staged block kernel, config 3 32.6 against 34.7 us
    // persistent, config 2 equal -- profiles/r02_exp/build_ab.txt)
    const bool persist_build = bsel == 3 || (bsel == 0 && bp.k <= 5 && !bp.vals64);
    // exact-fp64 fill: the persistent kernel (k <= 5) and the staged unrolled
    // block kernel (k in {1, 3, 5, 7, 11}); anything else builds tags only
    const bool unrolled = bp.k == 1 || bp.k == 3 || bp.k == 5 || bp.k == 7 || bp.k == 11;
    const bool f64_ok = bp.stage && unrolled && !warp_build &&
                        (persist_build ? bp.k <= 5 : (size_t)smem + (size_t)bp.stage_words * 8 <= 200 * 1024);
    if (!f64_ok) bp.vals64 = nullptr;
    *f64_done = bp.vals64 != nullptr;
    if (persist_build && bp.stage) {
        switch (bp.k) {
            case 1: return dense ? launch_p<1, true>(bp, st) : launch_p<1, false>(bp, st);
            case 3: return dense ? launch_p<3, true>(bp, st) : launch_p<3, false>(bp, st);
            case 5: return dense ? launch_p<5, true>(bp, st) : launch_p<5, false>(bp, st);
            case 7: return dense ? launch_p<7, true>(bp, st) : launch_p<7, false>(bp, st);
            default: break;
        }
    }
    if (warp_build) {
        switch (bp.k) {
            case 1: return dense ? launch_w<1, true>(bp, st) : launch_w<1, false>(bp, st);
            case 3: return dense ? launch_w<3, true>(bp, st) : launch_w<3, false>(bp, st);
            case 5: return dense ? launch_w<5, true>(bp, st) : launch_w<5, false>(bp, st);
            case 7: return dense ? launch_w<7, true>(bp, st) : launch_w<7, false>(bp, st);
            case 11: return dense ? launch_w<11, true>(bp, st) : launch_w<11, false>(bp, st);
            default: break;
        }
    }
    if (bp.stage) {  // the unrolled fill needs the staging area's K*K slots per row
        switch (bp.k) {
            case 1: return dense ? launch_k<1, true>(bp, block, smem, st) : launch_k<1, false>(bp, block, smem, st);
            case 3: return dense ? launch_k<3, true>(bp, block, smem, st) : launch_k<3, false>(bp, block, smem, st);
            case 5: return dense ? launch_k<5, true>(bp, block, smem, st) : launch_k<5, false>(bp, block, smem, st);
            case 7: return dense ? launch_k<7, true>(bp, block, smem, st) : launch_k<7, false>(bp, block, smem, st);
            case 11: return dense ? launch_k<11, true>(bp, block, smem, st) : launch_k<11, false>(bp, block, smem, st);
            default: break;
        }
    }
    return launch_k<0, false>(bp, block, smem, st);
}

// Exact-fp64 builds (spconv_build_transform_f64) run the fp32 build on tag
// taps (float)(q + 1) -- the structure then follows the DOUBLE taps' zero
// test, as inc/sparse.hpp:335 does -- and this pass swaps each tag for the
// tap's fp32 and fp64 values.  One streaming pass: 4 B read, 12 B written.
__global__ void __launch_bounds__(256) retag_kernel(float* vals, double* vals64, int64_t nnz, const float* t32,
                                                    const double* t64) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)vals[e] - 1;
        vals[e] = __ldg(t32 + q);
        __stcs(vals64 + e, __ldg(t64 + q));
    }
}

cudaError_t launch_retag(float* vals, double* vals64, int64_t nnz, const float* t32, const double* t64,
                         cudaStream_t st) {
    if (nnz <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (nnz + 255) / 256;
    const int grid = (int)(want < (int64_t)sms * 8 ? want : (int64_t)sms * 8);
    retag_kernel<<<grid, 256, 0, st>>>(vals, vals64, nnz, t32, t64);
    return cudaGetLastError();
}

}  // namespace spb
