#pragma once
// spmm_band.cuh -- the hot path (templates; instantiated per kernel side by
// band_k*.cu, dispatched by spmm_band.cu): SpMM of the conv transform T against an
// image-major batch, as two launches per call (check + apply, or the fused
// check-and-apply + its fixup pass; see 3. below).
//
// Contract (shared with spmm.cu): for every row of T,
//     acc = +0.0f; for e in row (column-ascending): acc = fmaf(val[e], x[col[e]], acc)
// -- the reference's row loop (inc/sparse.hpp:185-191) in fp32, bit-identical
// to oracle/spconv_oracle.c's spmv_f32_fma.
//
// 1. conv_band_check -- streams the whole CSR once per call (row_ptr, col_idx,
//    vals: the 8*nnz + 4*rows bytes the roofline charges) and decides, per
//    segment (one output image row x, TW consecutive output columns), whether
//    the stored rows are exactly the rows of the conv transform of the
//    handle's k x k taps: row (x, y) holds the taps (j, i) whose input pixel
//    (s x + j - p, s y + i - p) lies inside the image, at column
//    (s x + j - p) n + (s y + i - p), in (j, i) order, with value w[j][i].
//    A segment's rows are one contiguous run whose start and length are
//    closed-form: one warp per segment bulk-copies row_ptr and the run into
//    shared memory (no dependent load) and checks every row there -- interior
//    rows with an unrolled k*k compare, clipped rows over their tap range.
//    Result: one byte per segment (seg_ok).
//
// 2. conv_spmm_band -- register-blocked apply.  A CTA tile is TH output rows x
//    TW = 32*CPT output columns; each consumer thread owns V rows x CPT
//    adjacent columns.  Rows of T for vertically/horizontally adjacent pixels
//    share most of their columns (a k x k pattern shifted by s), so per input
//    row of its (s(V-1)+k) x (s(CPT-1)+k) receptive window a thread loads the
//    values ONCE (16-byte shared loads) and feeds every one of its V*CPT
//    outputs that stores that column: per output, k^2 FMAs and a fraction of a
//    shared load.  Input windows are staged by TMA 3-D box loads (cols x rows x
//    1 image; negative / out-of-range coordinates zero-fill = the padding),
//    STAGES deep, by a dedicated producer warp on full/empty mbarriers.  The
//    grid is persistent (one wave): work items (image, tile) are dealt
//    round-robin, image-major, so the CTAs sweep the batch together and window
//    halos shared by neighbouring tiles are L2 hits.  A warp whose rows all lie
//    in verified segments (and whose taps are finite and non-zero) takes the
//    blocked path; otherwise it runs the per-entry loop straight from the CSR.
//
// 3. Fused form (FUSED = true): the producer warp of each persistent CTA also
//    checks segments (same device functions as 1.) between its window loads;
//    the consumers take the blocked path unconditionally and conv_band_fixup
//    (a programmatic dependent) recomputes, from the CSR, the rows of any
//    segment that failed.  Used when the matrix is a small part of the call's
//    bytes; the host (capi.cu run_spmm) picks the form.
//
//    Blocked == per-entry, bit for bit: a tap that lands in the zero padding
//    executes fmaf(w, +0.0f, acc), which returns acc unchanged (w finite)
//    unless acc is exactly -0 -- reachable only when every earlier product
//    underflowed to -0 (|w*x| < 2^-150) -- where it may return +0 (DESIGN 8:
//    the sign of such a zero is the one bit-level exception).  So executing
//    or skipping the clipped taps is otherwise indistinguishable, and every
//    output still sees its stored taps in (j, i) = column-ascending order.
#include <algorithm>
#include <cstdlib>

#include "internal.h"
#include "tma.cuh"

namespace spb {

namespace {

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tap_range_dev(int x, int dim, int k, int s, int p, int& lo, int& hi) {
    lo = max(0, p - s * x);
    hi = min(k, dim + p - s * x);
    lo = min(lo, k);
    if (hi < lo) hi = lo;
}

// #{x' in [0, x) : tap index j lands inside the image at slide x'} (O(1)).
__device__ __forceinline__ int slides_before(int x, int j, int dim, int s, int p) {
    const int lo = (p - j <= 0) ? 0 : (p - j + s - 1) / s;
    const int hi = (dim + p - j - 1 < 0) ? 0 : (dim + p - j - 1) / s + 1;
    return max(0, min(x, hi) - lo);
}

constexpr int round_up(int v, int m) { return (v + m - 1) / m * m; }

// One stored entry of a row: fp32 fmaf (the device contract) or the
// reference's fp64 multiply then add, two roundings (inc/sparse.hpp:185-191).
__device__ __forceinline__ float band_step(float acc, float w, float x) { return fmaf(w, x, acc); }
__device__ __forceinline__ double band_step(double acc, double w, double x) { return __dadd_rn(acc, __dmul_rn(w, x)); }
constexpr int cmax(int a, int b) { return a > b ? a : b; }

}  // namespace

// ---------------------------------------------------------------------------
// Geometry of one instantiation.
// ---------------------------------------------------------------------------
// T: the element type of images and sums (float: the fp32 contract; double:
// the reference's own arithmetic, spconv_spmm_f64).
template <int K, int S, int V, int CPT, int TH, int STAGES, int DELTA, typename T = float>
struct BandCfg {
    static constexpr int E = 16 / (int)sizeof(T);       // elements per 16-byte vector
    // VEC: each thread's window columns start 16-byte aligned (s * CPT a
    // multiple of E) and are read with 16-byte shared loads; otherwise (s = 3)
    // element by element.
    static constexpr bool VEC = (S * CPT) % E == 0;
    static_assert(TH % V == 0, "TH must be a multiple of V");
    static constexpr int KK = K * K;
    static constexpr int TW = 32 * CPT;                 // output columns per tile
    static constexpr int NX = S * (CPT - 1) + K;        // window columns one thread reads per row
    static constexpr int NV4 = VEC ? (DELTA + NX + E - 1) / E : DELTA + NX;  // loads per row
    static constexpr int JJ = S * (V - 1) + K;          // window rows one thread reads
    static constexpr int WR = S * (TH - 1) + K;         // window rows
    static constexpr int WC = cmax(round_up(S * (TW - 1) + K + DELTA, 16 / (int)sizeof(T)),
                                   round_up(S * CPT * 31 + (VEC ? E : 1) * NV4, 16 / (int)sizeof(T)));
    static constexpr int WIN = WR * WC;
    static constexpr int CWARPS = TH / V;               // consumer warps
    static constexpr int THREADS = 32 * (CWARPS + 1);   // + one producer warp
    static constexpr int SF = round_up(WIN, 128 / (int)sizeof(T));  // elements per stage (128-byte aligned)
    static constexpr size_t SMEM = 128 + (size_t)STAGES * SF * sizeof(T);
    static_assert(WC <= 256 && WR <= 256, "TMA box limit");
    static_assert(TH <= 64, "at most two producer lanes per tile row");
    static_assert(STAGES * 24 <= 128, "barriers + flag masks fit the 128-byte header");
};

// ---------------------------------------------------------------------------
// 1. Band check: one warp per segment, everything it reads staged by bulk
//    copies issued before any of it is needed.
//
//    The segment's expected CSR footprint is closed-form (Theorem 2.1 prefix
//    sums): its rows start at S0 = CX(x) * SY + cx(x) * CY(y0) and hold
//    L = cx(x) * (CY(y0 + nr) - CY(y0)) entries, CX / CY being the running
//    per-slide tap counts.  So one elected lane issues three 1-D bulk copies
//    (row_ptr[r0 .. r0+nr], col_idx and vals over [S0, S0+L)) with no
//    dependent global load, and the warp then checks every row -- interior
//    rows with a fully unrolled k*k compare, clipped (border) rows with the
//    same compare over their tap range -- out of shared memory.  Rows of a
//    segment start at cx * (CY(y) - CY(y0)) inside the run.  If every
//    row_ptr matches its prediction and every entry matches the pattern, the
//    segment's rows are exactly the conv rows.  Result: one byte per segment.
// ---------------------------------------------------------------------------
// PER: most entries per major index (k^2 for CSR rows; ceil(k/s)^2 for CSC
// columns); SEG: majors per segment (TW output columns for CSR, TWC = s * TW
// input columns for CSC -- the same input footprint, so a CSC segment of the
// apply's tile width never holds more entries than a CSR one).
template <int K, int S, int TW, int PER = K * K, int SEG = TW>
struct CheckCfg {
    static constexpr int KK = K * K;
    static constexpr int TWC = S * TW;                     // CSC segment width (input columns)
    static constexpr int RUN = SEG * PER;                  // entries of a full segment
    static constexpr int BUFW = (RUN + 3 + 3) / 4 * 4;     // + alignment slack (16-byte bulk units)
    static constexpr int RPW = (TWC + 1 + 3 + 3) / 4 * 4;  // row_ptr / col_ptr words
    static constexpr int OFFW = S > 1 ? TWC : 0;           // CSC, s > 1: per-column run offsets
    static constexpr size_t WARP_BYTES = (size_t)(RPW + 2 * BUFW + OFFW) * 4;
    static_assert(SEG * PER <= TW * KK || SEG == TWC, "");
    // as many warps (<= 4) as fit 190 KB: k = 11 segments hold up to 121 entries per row
    static constexpr int WARPS = (190 * 1024) / WARP_BYTES >= 4 ? 4 : cmax(1, (int)((190 * 1024) / WARP_BYTES));
    static constexpr size_t SMEM = 128 + (size_t)WARPS * WARP_BYTES;
    static_assert(SMEM <= 200 * 1024, "segment too large for shared memory");
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Sum over slides x' < x of the taps landing inside [0, dim): CX(x) / CY(y).
template <int K, int S>
__device__ __forceinline__ int cum_taps(int x, int dim, int p) {
    int c = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) c += slides_before(x, j, dim, S, p);
    return c;
}

// One segment's closed-form footprint.
struct SegGeom {
    int x, y0, nr, r0, jlo, jhi, cy0, L;
    long long S0;
    bool valid;
};

// ZT: the taps include exact zeros (not stored; bit j*K+i of P.nzmask marks
// the non-zero ones).  The footprint is then the Theorem 2.1 prefix over the
// mask: S0 = sum_j W[j] * slides_before(x, j) + sum_i nzcol(i) * slides_before(y0, i)
// with W[j] = sum_i nz[j][i] * #{y : i lands}, nzcol(i) = sum_{j in J(x)} nz[j][i].
template <int K, int S, int TW, bool ZT>
__device__ __forceinline__ SegGeom seg_geom(const BandParams& P, long long seg) {
    SegGeom g;
    g.x = (int)(seg / P.tiles_y);
    g.y0 = (int)(seg - (long long)g.x * P.tiles_y) * TW;
    g.nr = min(TW, P.no - g.y0);
    g.r0 = g.x * P.no + g.y0;
    tap_range_dev(g.x, P.m, K, S, P.p, g.jlo, g.jhi);
    if (!ZT) {
        g.cy0 = cum_taps<K, S>(g.y0, P.n, P.p);
        g.S0 = (long long)cum_taps<K, S>(g.x, P.m, P.p) * P.sy + (long long)(g.jhi - g.jlo) * g.cy0;
        g.L = (g.jhi - g.jlo) * (cum_taps<K, S>(g.y0 + g.nr, P.n, P.p) - g.cy0);
    } else {
        const unsigned long long mk = P.nzmask;
        long long s0 = 0;
        int len = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) s0 += P.zw[j] * slides_before(g.x, j, P.m, S, P.p);
#pragma unroll
        for (int i = 0; i < K; ++i) {
            int nzc = 0;
#pragma unroll
            for (int j = 0; j < K; ++j) nzc += (j >= g.jlo && j < g.jhi && ((mk >> (j * K + i)) & 1ull)) ? 1 : 0;
            const int b0 = slides_before(g.y0, i, P.n, S, P.p);
            s0 += (long long)nzc * b0;
            len += nzc * (slides_before(g.y0 + g.nr, i, P.n, S, P.p) - b0);
        }
        g.cy0 = 0;
        g.S0 = s0;
        g.L = len;
    }
    g.valid = g.S0 + g.L <= (long long)P.nnz;  // (a matrix that is not this transform may run past the end)
    return g;
}

// Lane 0: the three bulk copies of a valid segment (row_ptr, col_idx, vals)
// into one staging slice of CheckCfg::WARP_BYTES, completing on `bar`.
template <int K, int S, int TW, int PER = K * K, int SEG = TW>
__device__ __forceinline__ void seg_issue(const BandParams& P, const SegGeom& g, int* rp, uint64_t* bar) {
    using C = CheckCfg<K, S, TW, PER, SEG>;
    int* cb = rp + C::RPW;
    int* vb = cb + C::BUFW;
    const int rbase = g.r0 & ~3;
    const uint32_t rwords = (uint32_t)((g.r0 + g.nr + 1 - rbase + 3) & ~3);
    const long long ebase = g.S0 & ~3ll;
    const uint32_t ewords = (uint32_t)((g.S0 + g.L - ebase + 3) & ~3ll);
    mbar_expect_tx(bar, 4u * (rwords + 2u * ewords));
    bulk_g2s(rp, P.row_ptr + rbase, 4u * rwords, bar);
    if (ewords) {
        bulk_g2s(cb, P.col_idx + ebase, 4u * ewords, bar);
        bulk_g2s(vb, P.vals + ebase, 4u * ewords, bar);
    }
}

// Whole warp, segment landed in the slice at `rp`: per-row offsets (a warp
// scan of cx * cy(y)), then every row checked from shared memory -- interior
// rows with the fully unrolled k*k compare, clipped rows over their tap
// range.  Returns the verdict (warp-uniform).
template <int K, int S, int TW, bool ZT>
__device__ __forceinline__ bool seg_verify(const BandParams& P, const SegGeom& g, const int* rp,
                                           const uint32_t (&w)[K * K], const uint32_t* s_w, int lane) {
    using C = CheckCfg<K, S, TW>;
    constexpr int RPL = TW / 32;  // rows per lane
    const int* cb = rp + C::RPW;
    const uint32_t* vb = reinterpret_cast<const uint32_t*>(cb + C::BUFW);
    const int cx = g.jhi - g.jlo;
    const unsigned long long mk = ZT ? P.nzmask : 0ull;
    int nzc[K];  // ZT: stored taps per tap column i over this segment's J(x)
#pragma unroll
    for (int i = 0; i < K; ++i) {
        nzc[i] = 0;
        if (ZT)
#pragma unroll
            for (int j = 0; j < K; ++j) nzc[i] += (j >= g.jlo && j < g.jhi && ((mk >> (j * K + i)) & 1ull)) ? 1 : 0;
    }
    int off[RPL], ilo_[RPL], ihi_[RPL];
    int run = 0;
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
        const int l = lane + 32 * q;
        tap_range_dev(g.y0 + l, P.n, K, S, P.p, ilo_[q], ihi_[q]);
        int rc = cx * (ihi_[q] - ilo_[q]);
        if (ZT) {
            rc = 0;
#pragma unroll
            for (int i = 0; i < K; ++i) rc += (i >= ilo_[q] && i < ihi_[q]) ? nzc[i] : 0;
        }
        const int c = l < g.nr ? rc : 0;
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        off[q] = run + inc - c;
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
    bool ok = run == g.L;
    const int* rps = rp + (g.r0 & 3);
    const int* cbs = cb + (int)(g.S0 & 3);
    const uint32_t* vbs = vb + (int)(g.S0 & 3);
    const int S0i = (int)g.S0;  // S0 + L <= nnz < 2^31 here
    uint32_t bad = 0;
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
        const int l = lane + 32 * q;
        if (l < g.nr) {
            const int y = g.y0 + l;
            ok &= rps[l] == S0i + off[q];
            if (l == g.nr - 1) ok &= rps[g.nr] == S0i + g.L;
            const int ilo = ilo_[q], ihi = ihi_[q];
            const int rb = (S * g.x - P.p) * P.n + (S * y - P.p);
            const int* cl = cbs + off[q];
            const uint32_t* vl = vbs + off[q];
            if (ZT) {  // stored taps only, in (j, i) order
                int e = 0;
                if (cx == K && ilo == 0 && ihi == K) {
                    // tap q sits at the popcount of the mask below it (row-invariant)
#pragma unroll
                    for (int j = 0; j < K; ++j)
#pragma unroll
                        for (int ii = 0; ii < K; ++ii) {
                            const int q = j * K + ii;
                            const int pos = __popcll(mk & ((1ull << q) - 1ull));
                            if ((mk >> q) & 1ull)
                                bad |= (uint32_t)(cl[pos] - (rb + j * P.n + ii)) | (vl[pos] ^ w[q]);
                        }
                } else {
                    for (int j = g.jlo; j < g.jhi; ++j)
                        for (int ii = ilo; ii < ihi; ++ii)
                            if ((mk >> (j * K + ii)) & 1ull) {
                                bad |= (uint32_t)(cl[e] - (rb + j * P.n + ii)) | (vl[e] ^ s_w[j * K + ii]);
                                ++e;
                            }
                }
            } else if (cx == K && ilo == 0 && ihi == K) {
#pragma unroll
                for (int j = 0; j < K; ++j)
#pragma unroll
                    for (int ii = 0; ii < K; ++ii)
                        bad |= (uint32_t)(cl[j * K + ii] - (rb + j * P.n + ii)) | (vl[j * K + ii] ^ w[j * K + ii]);
            } else {
                int e = 0;
                for (int j = g.jlo; j < g.jhi; ++j)
                    for (int ii = ilo; ii < ihi; ++ii, ++e)
                        bad |= (uint32_t)(cl[e] - (rb + j * P.n + ii)) | (vl[e] ^ s_w[j * K + ii]);
            }
        }
    }
    ok &= bad == 0u;
    return __all_sync(0xffffffffu, ok);
}

// ---------------------------------------------------------------------------
// 1b. The same check over CSC storage (inc/sparse.hpp:24-32: col_ptr, row_idx,
//     vals; csc_build.cu writes it).  Column c = (a, b) is input pixel (a, b);
//     it holds the outputs (x, y) with s x + j - p = a, s y + i - p = b for a
//     stored tap (j, i), rows ascending = j descending, then i descending.
//     A CSC segment is one input row a x TW consecutive input columns; its
//     entries are one contiguous run:
//        S0 = sum_j W[j] * #{x : 0 <= s x + j - p < a} + sum_i nzJ(i) * #{y : 0 <= s y + i - p < b0}
//        L  = sum_i nzJ(i) * #{y : b0 <= s y + i - p < b0 + nb}
//     with W[j] = sum_i nz[j][i] * #{y : tap i lands} (= sy for dense taps)
//     and nzJ(i) = #{stored (j, i) : j in J(a)} -- the closed form of
//     csc_build.cu's col_ptr.  The same three bulk copies stage col_ptr and
//     the run, and every column is compared with the taps landing on it.
// ---------------------------------------------------------------------------

// #{x in [0, mo) : 0 <= s x + j - p < a}: slides of tap row j that read an input row above a.
__device__ __forceinline__ int slides_below(int j, int a, int mo, int s, int p) {
    if (a <= 0) return 0;
    const int lo = p - j <= 0 ? 0 : (p - j + s - 1) / s;  // s x >= p - j
    const int b = a - 1 + p - j;                            // s x <= a - 1 + p - j
    if (b < 0) return 0;
    const int hi = min(mo - 1, b / s);
    return max(0, hi - lo + 1);
}

// Bit j: tap row j lands on input row a for some output row x in [0, mo).
template <int K, int S>
__device__ __forceinline__ uint32_t tap_set_mask(int a, int mo, int p) {
    uint32_t mk = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int d = a + p - j;
        if (d >= 0 && d % S == 0 && d / S < mo) mk |= 1u << j;
    }
    return mk;
}

// Stored taps of row j as K bits (bit i).
template <int K, bool ZT>
__device__ __forceinline__ uint32_t nz_row(unsigned long long nzmask, int j) {
    return ZT ? (uint32_t)((nzmask >> (j * K)) & ((1ull << K) - 1ull)) : ((1u << K) - 1u);
}

// TW here = the CSC segment width (CheckCfg::TWC).
template <int K, int S, int TW, bool ZT>
__device__ __forceinline__ SegGeom seg_geom_csc(const BandParams& P, long long seg) {
    SegGeom g;
    g.x = (int)(seg / P.tiles_b);                                 // input row a
    g.y0 = (int)(seg - (long long)g.x * P.tiles_b) * TW;          // first input column b0
    g.nr = min(TW, P.n - g.y0);
    g.r0 = g.x * P.n + g.y0;                                      // first column index
    const uint32_t jm = tap_set_mask<K, S>(g.x, P.mo, P.p);
    g.jlo = (int)jm;  // (the J(a) mask)
    g.jhi = 0;
    long long s0 = 0;
    int len = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) s0 += (ZT ? P.zw[j] : (long long)P.sy) * slides_below(j, g.x, P.mo, S, P.p);
#pragma unroll
    for (int i = 0; i < K; ++i) {
        int nzj = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) nzj += ((jm >> j) & 1u) && ((nz_row<K, ZT>(P.nzmask, j) >> i) & 1u) ? 1 : 0;
        const int b0 = slides_below(i, g.y0, P.no, S, P.p);
        s0 += (long long)nzj * b0;
        len += nzj * (slides_below(i, g.y0 + g.nr, P.no, S, P.p) - b0);
    }
    g.cy0 = 0;
    g.S0 = s0;
    g.L = len;
    g.valid = g.S0 + g.L <= (long long)P.nnz;
    return g;
}

// Whole warp, CSC segment landed at `rp` (col_ptr words, then row_idx, vals):
// per-column offsets by a warp scan of the column counts, col_ptr compared,
// then each column's rows and values compared with the taps that land on it
// (interior stride-1 columns of dense taps fully unrolled).
// Interior CSC column of residue class (RA, RB) = (a + p, b + p) mod s: all
// NJ x NI taps of the class land; rows r0 + dj * n_out + di, taps (JT - s dj, IT - s di).
template <int K, int S, int RA, int RB>
__device__ __forceinline__ uint32_t csc_interior(const int* cl, const uint32_t* vl, int a, int b, int p, int no,
                                                 const uint32_t (&w)[K * K]) {
    constexpr int NJ = (K - 1 - RA) / S + 1, JT = RA + S * (NJ - 1);
    constexpr int NI = (K - 1 - RB) / S + 1, IT = RB + S * (NI - 1);
    const int r0 = (a + p - JT) / S * no + (b + p - IT) / S;
    uint32_t bad = 0;
#pragma unroll
    for (int dj = 0; dj < NJ; ++dj)
#pragma unroll
        for (int di = 0; di < NI; ++di)
            bad |= (uint32_t)(cl[dj * NI + di] - (r0 + dj * no + di)) | (vl[dj * NI + di] ^ w[(JT - S * dj) * K + (IT - S * di)]);
    return bad;
}

// #{i in [0, K) : i == rb (mod S), 0 <= (b + p - i) / S < no}: the taps landing on input column b.
template <int K, int S>
__device__ __forceinline__ int taps_on(int b, int p, int no) {
    const int bp = b + p;
    const int lo = max(0, bp - S * (no - 1)), hi = min(K - 1, bp);
    const int first = lo + (((bp - lo) % S) + S) % S;  // first i >= lo with i == bp (mod S)
    return first > hi ? 0 : (hi - first) / S + 1;
}

// (s = 1 in the fused producer's staging layout, CheckCfg<K, 1, TW>)
template <int K, int S, int TW, bool ZT>
__device__ __forceinline__ bool seg_verify_csc_s1(const BandParams& P, const SegGeom& g, const int* rp,
                                               const uint32_t (&w)[K * K], const uint32_t* s_w, int lane) {
    using C = CheckCfg<K, S, TW>;
    constexpr int RPL = TW / 32;  // columns per lane
    const int* cb = rp + C::RPW;
    const uint32_t* vb = reinterpret_cast<const uint32_t*>(cb + C::BUFW);
    const uint32_t jm = (uint32_t)g.jlo;
    const int a = g.x;
    int off[RPL];
    uint32_t im_[RPL];
    int run = 0;
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
        const int l = lane + 32 * q;
        const uint32_t im = tap_set_mask<K, S>(g.y0 + l, P.no, P.p);
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < K; ++j)
            if ((jm >> j) & 1u) cnt += __popc(nz_row<K, ZT>(P.nzmask, j) & im);
        im_[q] = im;
        const int c = l < g.nr ? cnt : 0;
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        off[q] = run + inc - c;
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
    bool ok = run == g.L;
    const int* rps = rp + (g.r0 & 3);
    const int* cbs = cb + (int)(g.S0 & 3);
    const uint32_t* vbs = vb + (int)(g.S0 & 3);
    const int S0i = (int)g.S0;
    constexpr uint32_t FULL = (1u << K) - 1u;
    uint32_t bad = 0;
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
        const int l = lane + 32 * q;
        if (l < g.nr) {
            const int b = g.y0 + l;
            ok &= rps[l] == S0i + off[q];
            if (l == g.nr - 1) ok &= rps[g.nr] == S0i + g.L;
            const uint32_t im = im_[q];
            const int* cl = cbs + off[q];
            const uint32_t* vl = vbs + off[q];
            if (!ZT && S == 1 && jm == FULL && im == FULL) {
                // every tap lands: rows (a + p - j, b + p - i) for j, i descending
                const int rb = (a + P.p - (K - 1)) * P.no + (b + P.p - (K - 1));
#pragma unroll
                for (int jj = 0; jj < K; ++jj)
#pragma unroll
                    for (int ii = 0; ii < K; ++ii)
                        bad |= (uint32_t)(cl[jj * K + ii] - (rb + jj * P.no + ii)) |
                               (vl[jj * K + ii] ^ w[(K - 1 - jj) * K + (K - 1 - ii)]);
            } else {
                int e = 0;
#pragma unroll
                for (int j = K - 1; j >= 0; --j) {
                    if (!((jm >> j) & 1u)) continue;
                    const int xrow = (a + P.p - j) / S * P.no;
                    const uint32_t cm = nz_row<K, ZT>(P.nzmask, j) & im;
#pragma unroll
                    for (int i = K - 1; i >= 0; --i) {
                        if (!((cm >> i) & 1u)) continue;
                        bad |= (uint32_t)(cl[e] - (xrow + (b + P.p - i) / S)) | (vl[e] ^ s_w[j * K + i]);
                        ++e;
                    }
                }
            }
        }
    }
    ok &= bad == 0u;
    return __all_sync(0xffffffffu, ok);
}

template <int K, int S, int TW, bool ZT, int PER = K * K, int SEG = TW>
__device__ __forceinline__ bool seg_verify_csc(const BandParams& P, const SegGeom& g, int* rp,
                                               const uint32_t (&w)[K * K], const uint32_t* s_w, int lane) {
    using C = CheckCfg<K, S, TW, PER, SEG>;
    if constexpr (S == 1 && PER == K * K) return seg_verify_csc_s1<K, S, TW, ZT>(P, g, rp, w, s_w, lane);
    constexpr int TWC = C::TWC;
    constexpr int RPL = TWC / 32;  // columns per lane
    const int* cb = rp + C::RPW;
    const uint32_t* vb = reinterpret_cast<const uint32_t*>(cb + C::BUFW);
    const uint32_t jm = (uint32_t)g.jlo;
    const int a = g.x;
    const int nj = __popc(jm);
    const int* rps = rp + (g.r0 & 3);
    const int S0i = (int)g.S0;
    const int* cbs = cb + (int)(g.S0 & 3);
    const uint32_t* vbs = vb + (int)(g.S0 & 3);
    // 1. column counts in natural order: warp scan -> offsets; col_ptr compared
    int run = 0, off[RPL];
    uint32_t im_[RPL];  // (s = 1: the column tap masks, kept for pass 2)
    bool ok = true;
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
        const int l = lane + 32 * q;
        int cnt = 0;
        if (ZT || S == 1) {
            const uint32_t im = tap_set_mask<K, S>(g.y0 + l, P.no, P.p);
            im_[q] = im;
#pragma unroll
            for (int j = 0; j < K; ++j)
                if ((jm >> j) & 1u) cnt += __popc(nz_row<K, ZT>(P.nzmask, j) & im);
        } else {
            cnt = nj * taps_on<K, S>(g.y0 + l, P.p, P.no);
        }
        const int c = l < g.nr ? cnt : 0;
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        off[q] = run + inc - c;
        if (l < g.nr) {
            ok &= rps[l] == S0i + off[q];
            if (l == g.nr - 1) ok &= rps[g.nr] == S0i + g.L;
        }
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
    ok &= run == g.L;
    uint32_t bad = 0;
    if constexpr (S >= 3 && !ZT) {
        // Interior segment (every column receives every tap of its residue
        // class): the run is periodic -- S consecutive columns hold
        // D = NJ * K entries, and the next S columns the same taps on rows
        // one output column further.  Each lane owns fixed positions r of a
        // block of G periods (its expected row offset and tap computed once),
        // and the warp walks the run in blocks: consecutive lanes read
        // consecutive words (no bank conflicts, unlike a lane per column).
        // s = 3 (k7: 326 -> 243 us at 2048^2 x 32 images); s = 2 keeps the
        // residue-uniform unrolled compares below, which measured faster
        // (config 4: 546 against 589 us, scripts/probe_csc_check.py).
        const int ra = (a + P.p) % S, NJ = (K - 1 - ra) / S + 1;
        bool inter = nj == NJ && g.nr == TWC;
#pragma unroll
        for (int c = 0; c < S; ++c) {
            const int bl = g.y0 + c, bh = g.y0 + TWC - S + c;
            inter &= taps_on<K, S>(bl, P.p, P.no) == (K - 1 - (bl + P.p) % S) / S + 1;
            inter &= taps_on<K, S>(bh, P.p, P.no) == (K - 1 - (bh + P.p) % S) / S + 1;
        }
        if (inter) {
            constexpr int DMAX = ((K + S - 1) / S) * K;
            constexpr int UC = DMAX > 64 ? (DMAX + 31) / 32 : 2;
            const int D = NJ * K;
            const int G = cmax(1, 32 * UC / D);
            const int JT = ra + S * (NJ - 1);
            const int xr = (a + P.p - JT) / S;
            int rowu[UC], ru[UC], gpu[UC];
            uint32_t tapu[UC];
#pragma unroll
            for (int u = 0; u < UC; ++u) {
                const int r = lane + 32 * u;
                const int gp = r / D, rr = r - gp * D;
                // the period's column holding position rr (columns in order from
                // the segment's first, each with NJ * NI(residue) entries)
                int cp = S - 1, eb = 0, ni = 1, it = 0, e0 = 0;
                bool found = false;
#pragma unroll
                for (int c = 0; c < S; ++c) {
                    const int rb = (g.y0 + c + P.p) % S;
                    const int n_i = (K - 1 - rb) / S + 1;
                    if (!found && rr < e0 + NJ * n_i) {
                        found = true;
                        cp = c;
                        ni = n_i;
                        it = rb + S * (n_i - 1);
                        eb = e0;
                    }
                    e0 += NJ * n_i;
                }
                const int kk = rr - eb;
                const int dj = kk / ni, di = kk - dj * ni;
                ru[u] = r < G * D ? r : -1;
                gpu[u] = gp;
                rowu[u] = (xr + dj) * P.no + (g.y0 + cp + P.p - it) / S + gp + di;
                tapu[u] = s_w[(JT - S * dj) * K + (it - S * di)];
            }
            const int full = (TW / G) * G;  // periods in whole blocks
            const int step = G * D;
            int g0 = 0, base = 0;
#pragma unroll 1
            for (; g0 < full; g0 += G, base += step) {
#pragma unroll
                for (int u = 0; u < UC; ++u)
                    if (ru[u] >= 0)
                        bad |= (uint32_t)(cbs[base + ru[u]] - (rowu[u] + g0)) | (vbs[base + ru[u]] ^ tapu[u]);
            }
#pragma unroll
            for (int u = 0; u < UC; ++u)  // the last, partial block
                if (ru[u] >= 0 && g0 + gpu[u] < TW)
                    bad |= (uint32_t)(cbs[base + ru[u]] - (rowu[u] + g0)) | (vbs[base + ru[u]] ^ tapu[u]);
            ok &= bad == 0u;
            return __all_sync(0xffffffffu, ok);
        }
    }
    if constexpr (S == 1) {
        // 2. every column's rows and values against the taps landing on it
        //    (interior columns of dense taps fully unrolled)
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            const int l = lane + 32 * q;
            if (l >= g.nr) continue;
            const int b = g.y0 + l;
            const int* cl = cbs + off[q];
            const uint32_t* vl = vbs + off[q];
            const uint32_t im = im_[q];
            if (!ZT && jm == (1u << K) - 1u && im == (1u << K) - 1u) {
                const int rb = (a + P.p - (K - 1)) * P.no + (b + P.p - (K - 1));
#pragma unroll
                for (int jj = 0; jj < K; ++jj)
#pragma unroll
                    for (int ii = 0; ii < K; ++ii)
                        bad |= (uint32_t)(cl[jj * K + ii] - (rb + jj * P.no + ii)) |
                               (vl[jj * K + ii] ^ w[(K - 1 - jj) * K + (K - 1 - ii)]);
            } else {
                int e = 0;
#pragma unroll
                for (int j = K - 1; j >= 0; --j) {
                    if (!((jm >> j) & 1u)) continue;
                    const int xrow = (a + P.p - j) * P.no;
                    const uint32_t cm = nz_row<K, ZT>(P.nzmask, j) & im;
#pragma unroll
                    for (int i = K - 1; i >= 0; --i) {
                        if (!((cm >> i) & 1u)) continue;
                        bad |= (uint32_t)(cl[e] - (xrow + (b + P.p - i))) | (vl[e] ^ s_w[j * K + i]);
                        ++e;
                    }
                }
            }
        }
    } else if constexpr (S >= 3) {
        // 2. s >= 3: every column with the taps' loop (few entries per column)
#pragma unroll 1
        for (int q = 0; q < RPL; ++q) {
            const int l = lane + 32 * q;
            if (l >= g.nr) continue;
            const int b = g.y0 + l;
            const int* cl = cbs + off[q];
            const uint32_t* vl = vbs + off[q];
            const uint32_t im = tap_set_mask<K, S>(b, P.no, P.p);
            int e = 0;
#pragma unroll 1
            for (int j = K - 1; j >= 0; --j) {
                if (!((jm >> j) & 1u)) continue;
                const int xrow = (a + P.p - j) / S * P.no;
                const uint32_t cm = nz_row<K, ZT>(P.nzmask, j) & im;
#pragma unroll 1
                for (int i = K - 1; i >= 0; --i) {
                    if (!((cm >> i) & 1u)) continue;
                    bad |= (uint32_t)(cl[e] - (xrow + (b + P.p - i) / S)) | (vl[e] ^ s_w[j * K + i]);
                    ++e;
                }
            }
        }
    } else {
        // 2. s = 2: lanes in residue-uniform order (pass q covers columns
        //    b0 + s * lane + (q mod s) of its group), so every lane of a pass
        //    has the same interior tap pattern: one warp-uniform branch.
        int* s_off = rp + C::RPW + 2 * C::BUFW;
#pragma unroll
        for (int q = 0; q < RPL; ++q) s_off[lane + 32 * q] = off[q];
        __syncwarp();
        const int ra = (a + P.p) % S, NJ = (K - 1 - ra) / S + 1;
#pragma unroll 1
        for (int q = 0; q < RPL; ++q) {
            const int l = (q / S) * 32 * S + S * lane + (q % S);
            const int b = g.y0 + l;
            const int rb = (b + P.p) % S;  // (warp-uniform)
            const int o = s_off[l];
            const int* cl = cbs + o;
            const uint32_t* vl = vbs + o;
            const bool live = l < g.nr;
            const bool interior = !ZT && nj == NJ && taps_on<K, S>(b, P.p, P.no) == (K - 1 - rb) / S + 1;
            if (live && interior) {
                const int pat = ra * S + rb;
                if (pat == 0)
                    bad |= csc_interior<K, S, 0, 0>(cl, vl, a, b, P.p, P.no, w);
                else if (pat == 1)
                    bad |= csc_interior<K, S, 0, 1>(cl, vl, a, b, P.p, P.no, w);
                else if (pat == 2)
                    bad |= csc_interior<K, S, 1, 0>(cl, vl, a, b, P.p, P.no, w);
                else
                    bad |= csc_interior<K, S, 1, 1>(cl, vl, a, b, P.p, P.no, w);
            } else if (live) {
                const uint32_t im = tap_set_mask<K, S>(b, P.no, P.p);
                int e = 0;
#pragma unroll 1
                for (int j = K - 1; j >= 0; --j) {
                    if (!((jm >> j) & 1u)) continue;
                    const int xrow = (a + P.p - j) / S * P.no;
                    const uint32_t cm = nz_row<K, ZT>(P.nzmask, j) & im;
#pragma unroll 1
                    for (int i = K - 1; i >= 0; --i) {
                        if (!((cm >> i) & 1u)) continue;
                        bad |= (uint32_t)(cl[e] - (xrow + (b + P.p - i) / S)) | (vl[e] ^ s_w[j * K + i]);
                        ++e;
                    }
                }
            }
        }
    }
    ok &= bad == 0u;
    return __all_sync(0xffffffffu, ok);
}

// (CSC: the staging is sized for ceil(k/s)^2 entries per column)
template <int K, int S, int TW>
constexpr int csc_per() { return ((K + S - 1) / S) * ((K + S - 1) / S); }

template <int K, int S, int TW, bool ZT, bool CSCM>
__global__ void __launch_bounds__(128) conv_band_check(const BandParams P) {
    constexpr int PER = CSCM ? csc_per<K, S, TW>() : K * K;
    constexpr int SEG = CSCM ? S * TW : TW;
    using C = CheckCfg<K, S, TW, PER, SEG>;
    constexpr int KK = K * K;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t s_w[KK];  // taps, runtime-indexed (clipped rows)
    for (int q = threadIdx.x; q < KK; q += blockDim.x) s_w[q] = __float_as_uint(__ldg(P.taps + q));

    const long long seg = (long long)blockIdx.x * C::WARPS + warp;
    constexpr bool csc = CSCM;
    const bool live = seg < (csc ? (long long)P.m * P.tiles_b : (long long)P.mo * P.tiles_y);  // warp-uniform
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + warp;
    int* rp = reinterpret_cast<int*>(smem + 128 + (size_t)warp * C::WARP_BYTES);
    SegGeom g{};
    if (live) {
        g = csc ? seg_geom_csc<K, S, S * TW, ZT>(P, seg) : seg_geom<K, S, TW, ZT>(P, seg);
        if (lane == 0) {
            mbar_init(bar, 1);
            mbar_fence_init();
            if (g.valid) seg_issue<K, S, TW, PER, SEG>(P, g, rp, bar);
        }
    }
    __syncthreads();  // s_w (and the barrier inits) visible block-wide
    // (as a programmatic dependent: the matrix and taps are read early, the
    // flags -- which the kernel in front may still read -- written after it)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (!live) return;
    if (!g.valid) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (lane == 0) {
            P.seg_ok[seg] = 0;
            if (csc) *P.fail_count = 1;
        }
        return;
    }
    uint32_t w[KK];  // taps, compile-time indexed (full rows)
#pragma unroll
    for (int q = 0; q < KK; ++q) w[q] = s_w[q];
    mbar_wait(bar, 0);
    const bool ok = csc ? seg_verify_csc<K, S, TW, ZT, PER, SEG>(P, g, rp, w, s_w, lane)
                        : seg_verify<K, S, TW, ZT>(P, g, rp, w, s_w, lane);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (lane == 0) {
        P.seg_ok[seg] = ok ? 1 : 0;
        if (csc && !ok) *P.fail_count = 1;
    }
}

// ---------------------------------------------------------------------------
// 2. Register-blocked apply.
// ---------------------------------------------------------------------------

// Persistent work walk: item i = img * tiles + tx * tiles_y + ty, visited as
// i = blockIdx.x, blockIdx.x + gridDim.x, ... with the mixed-radix step
// precomputed once (no per-item division).
struct ItemIter {
    int img, tx, ty;
    int s_img, s_tx, s_ty, tiles_x, tiles_y;
    __device__ explicit ItemIter(const BandParams& P) {
        tiles_y = P.tiles_y;
        tiles_x = P.tiles / P.tiles_y;
        int t = (int)(blockIdx.x % (unsigned)P.tiles);
        img = (int)(blockIdx.x / (unsigned)P.tiles);
        tx = t / tiles_y;
        ty = t - tx * tiles_y;
        t = (int)(gridDim.x % (unsigned)P.tiles);
        s_img = (int)(gridDim.x / (unsigned)P.tiles);
        s_tx = t / tiles_y;
        s_ty = t - s_tx * tiles_y;
    }
    __device__ void next() {
        ty += s_ty;
        tx += s_tx;
        img += s_img;
        if (ty >= tiles_y) ty -= tiles_y, ++tx;
        if (tx >= tiles_x) tx -= tiles_x, ++img;
    }
};
// FUSED: one kernel does the band check and the apply.  The producer warp,
// between window loads, checks segments blockIdx.x, blockIdx.x + gridDim.x,
// ... (bulk copies double-buffered in two extra staging slices), and the
// consumers take the blocked path unconditionally; conv_band_fixup, launched
// right after on the same stream, recomputes the rows of any segment that
// failed its check from the CSR (normally none: it only reads the flags).
// ZT: some taps are exact zeros.  The blocked sums still run over all k*k
// taps: for a finite x, fmaf(0, x, acc) == acc (up to the sign of a zero acc,
// see the header), so they equal the stored-taps sums; a thread whose sums are
// not all finite (a non-finite x it read, where 0 * inf would differ) redoes
// its outputs per entry from the CSR.
// One stage's window (WR rows x WC columns of image `img`, starting at input
// row wr0, column wc0; out-of-image elements zero = the padding), loaded into
// shared memory.  TMA (one elected lane, one 3-D box) when the rows are
// 16-byte pitched; otherwise (P.notma: odd widths, s = 3 windows wider than a
// box) every producer lane issues cp.async element copies -- zero-filled out
// of the image -- whose completion each lane hands to the stage's `full`
// mbarrier (initialised for 32 + 1 arrivals in that mode).
template <typename C, typename T>
__device__ __forceinline__ void load_window(const BandParams& P, const CUtensorMap* tmap, T* dst, int wc0, int wr0,
                                            int img, uint64_t* full, int lane) {
    if (!P.notma) {
        if (lane == 0) {
            mbar_expect_tx(full, (uint32_t)(C::WIN * sizeof(T)));
            tma_load_3d(dst, tmap, wc0, wr0, img, full);
        }
        return;
    }
    const T* X = reinterpret_cast<const T*>(P.X) + (long long)img * P.ldx;
    // Row by row (the row's bounds and base pointer once), the row's columns
    // unrolled: a few instructions per element copy -- the producer warp's
    // issue rate is what feeds the consumers in this mode (k11 on 257 x 193:
    // ~30 instructions an element with a div/mod per element starved them).
    const uint32_t d0 = smem_u32(dst);
    const unsigned m = (unsigned)P.m, n = (unsigned)P.n;
#pragma unroll 1
    for (int r = 0; r < C::WR; ++r) {
        const int gr = wr0 + r;
        const bool rin = (unsigned)gr < m;
        const T* srow = X + (long long)(rin ? gr : 0) * P.n;
        const uint32_t drow = d0 + (uint32_t)(r * C::WC * sizeof(T));
#pragma unroll
        for (int c0 = 0; c0 < C::WC; c0 += 32) {
            const int c = c0 + lane;
            if (C::WC % 32 != 0 && c >= C::WC) break;
            const int gc = wc0 + c;
            const bool in = rin && (unsigned)gc < n;
            const T* src = in ? srow + gc : X;
            if constexpr (sizeof(T) == 4)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(drow + 4u * (uint32_t)c), "l"(src),
                             "r"(in ? 4 : 0)
                             : "memory");
            else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(drow + 8u * (uint32_t)c), "l"(src),
                             "r"(in ? 8 : 0)
                             : "memory");
        }
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full)) : "memory");
    // (+ one ordinary arrive: releases lane 0's earlier shared stores, the row flags)
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(full)) : "memory");
}

// The fused form: besides the consumers and the window producer, CHK warps
// check segments (two staging slices each, double-buffered), as many as the
// shared memory left by the window stages holds (<= 4; 0: no fused form).
template <int K, int S, int V, int CPT, int TH, int STAGES, int DELTA, typename T = float>
struct FusedCfg {
    using C = BandCfg<K, S, V, CPT, TH, STAGES, DELTA, T>;
    using CC = CheckCfg<K, S, C::TW>;
    static constexpr size_t HDR = 256;  // mbarriers, row flags, 2 x CHK check barriers
    static constexpr size_t BASE = HDR + (size_t)STAGES * C::SF * sizeof(T);
    static constexpr long long FREE = 227ll * 1024 - (long long)BASE;
    static constexpr int CHK = FREE <= 0 ? 0 : (FREE / (2 * (long long)CC::WARP_BYTES) >= 4 ? 4 : (int)(FREE / (2 * (long long)CC::WARP_BYTES)));
    static constexpr size_t SMEM = BASE + (size_t)CHK * 2 * CC::WARP_BYTES;
    static constexpr int THREADS = C::THREADS + 32 * CHK;
    static_assert(STAGES * 24 + 16 * 4 <= (int)HDR, "barriers fit the header");
};

template <int K, int S, int V, int CPT, int TH, int STAGES, int DELTA, bool FUSED, bool ZT = false,
          typename T = float>
__global__ void __launch_bounds__(FUSED ? FusedCfg<K, S, V, CPT, TH, STAGES, DELTA, T>::THREADS
                                        : BandCfg<K, S, V, CPT, TH, STAGES, DELTA, T>::THREADS,
                                  1)
    conv_spmm_band(const __grid_constant__ CUtensorMap tmap, const BandParams P) {
    using C = BandCfg<K, S, V, CPT, TH, STAGES, DELTA, T>;
    using CC = CheckCfg<K, S, C::TW>;
    using FC = FusedCfg<K, S, V, CPT, TH, STAGES, DELTA, T>;
    constexpr int CHK = FUSED ? FC::CHK : 0;
    constexpr size_t HDR = FUSED ? FC::HDR : 128;
    constexpr bool F64 = sizeof(T) == 8;
    static_assert(!FUSED || !F64, "the fp64 apply runs after a separate check");
    static_assert(!FUSED || CHK > 0, "no room for check warps");
    static_assert(FUSED || STAGES * 24 <= 128, "barriers fit the header");
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + STAGES;
    unsigned long long* s_mask = reinterpret_cast<unsigned long long*>(empty + STAGES);  // per-stage row flags
    uint64_t* cbar = reinterpret_cast<uint64_t*>(s_mask + STAGES);                       // (FUSED) check slices
    T* xs = reinterpret_cast<T*>(smem + HDR);
    __shared__ uint32_t s_w[C::KK];  // taps, runtime-indexed (checks, the CSC per-entry loop)
    __shared__ T s_wt[C::KK];        // the taps the sums use (fp64: the exact taps)

    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;

    if (t == 0) {
        tma_prefetch_desc(&tmap);
        for (int st = 0; st < STAGES; ++st) {
            mbar_init(&full[st], P.notma ? 33 : 1);
            mbar_init(&empty[st], C::CWARPS);
        }
        for (int b = 0; b < 2 * CHK; ++b) mbar_init(&cbar[b], 1);
        mbar_fence_init();
    }
    for (int q = t; q < C::KK; q += blockDim.x) {
        const float t32 = __ldg(P.taps + q);
        s_w[q] = __float_as_uint(t32);
        s_wt[q] = F64 && P.taps64 ? (T)__ldg(P.taps64 + q) : (T)t32;
    }
    __syncthreads();
    // Programmatic dependent launch: the next call's CTAs may start as SMs free
    // up.  What this grid reads before griddepcontrol.wait is the matrix and
    // the taps only (never written by the previous kernel: the host launches it
    // this way only after the handle's build and when its storage was never
    // handed out); X, Y, the row flags and the verdicts wait.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (FUSED && warp > C::CWARPS) {
        // ---- check warps (fused form): segments blockIdx.x * CHK + cw,
        // + gridDim.x * CHK, ..., two staging slices each: the copies of the
        // next segment are in flight while the current one is verified.
        const int cw = warp - C::CWARPS - 1;
        uint32_t w[C::KK];
#pragma unroll
        for (int q = 0; q < C::KK; ++q) w[q] = s_w[q];
        constexpr int SLICE = (int)(CC::WARP_BYTES / 4);
        int* cslice = reinterpret_cast<int*>(smem + HDR + (size_t)STAGES * C::SF * sizeof(T)) + 2 * cw * SLICE;
        uint64_t* bars = cbar + 2 * cw;
        const bool csc = P.csc != 0;
        const long long nseg = csc ? (long long)P.m * P.tiles_b : (long long)P.mo * P.tiles_y;
        const long long step = (long long)gridDim.x * CHK;
        long long cseg = (long long)blockIdx.x * CHK + cw;
        SegGeom vg{};
        int cb = 0;
        uint32_t cph = 0;
        bool waited = false;
        auto issue = [&](long long sg) {
            vg = csc ? seg_geom_csc<K, S, S * C::TW, ZT>(P, sg) : seg_geom<K, S, C::TW, ZT>(P, sg);
            if (lane == 0 && vg.valid) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                seg_issue<K, S, C::TW>(P, vg, cslice + cb * SLICE, &bars[cb]);
            }
        };
        if (cseg < nseg) issue(cseg);
        while (cseg < nseg) {
            const SegGeom g = vg;
            const long long sg = cseg;
            const int b = cb;
            cb ^= 1;
            cseg += step;
            __syncwarp();  // slice cb's previous segment was fully read before its verdict
            if (cseg < nseg) issue(cseg);
            bool ok = false;
            if (g.valid) {
                mbar_wait(&bars[b], (cph >> b) & 1u);
                cph ^= 1u << b;
                ok = csc ? seg_verify_csc<K, S, C::TW, ZT>(P, g, cslice + b * SLICE, w, s_w, lane)
                         : seg_verify<K, S, C::TW, ZT>(P, g, cslice + b * SLICE, w, s_w, lane);
            }
            if (!waited) {  // (the previous kernel may still read the flags)
                asm volatile("griddepcontrol.wait;" ::: "memory");
                waited = true;
            }
            if (lane == 0) {
                P.seg_ok[sg] = ok ? 1 : 0;
                if (!ok && !P.fixup) *P.fail_count = 1;
            }
        }
        return;
    }

    if (warp == C::CWARPS) {
        // ---- producer warp: per item, the tile rows' band-check flags (one
        // lane per row, folded into a per-stage bit mask) and the window load
        // (one elected lane).  Running STAGES items ahead hides the flag
        // loads' latency from the consumers.
        asm volatile("griddepcontrol.wait;" ::: "memory");
        int it = 0;
        for (ItemIter I(P); I.img < P.batch; I.next(), ++it) {
            const int st = it % STAGES;
            unsigned long long rows_ok = ~0ull;
            if (!FUSED && !P.csc) {  // (CSC / fused: the apply does not wait for per-row verdicts)
              rows_ok = 0;
#pragma unroll
              for (int h = 0; h < (TH + 31) / 32; ++h) {  // one lane per tile row
                bool f = true;
                if (32 * h + lane < TH) {
                    const int x = I.tx * TH + 32 * h + lane;
                    // (the check's segments are TW / seg_div columns wide)
                    for (int d = 0; d < P.seg_div && x < P.mo; ++d) {
                        const int sg = I.ty * P.seg_div + d;
                        if (sg < P.tiles_y_chk) f &= __ldg(P.seg_ok + (long long)x * P.tiles_y_chk + sg) != 0;
                    }
                }
                rows_ok |= (unsigned long long)__ballot_sync(0xffffffffu, f) << (32 * h);
              }
            }
            if (lane == 0) {
                if (it >= STAGES) mbar_wait(&empty[st], (uint32_t)(((it / STAGES) - 1) & 1));
                s_mask[st] = rows_ok;
            }
            __syncwarp();  // (the stage is free before any lane copies into it)
            load_window<C, T>(P, &tmap, xs + (size_t)st * C::SF, S * I.ty * C::TW - P.p - DELTA, S * I.tx * TH - P.p,
                              I.img, &full[st], lane);
            __syncwarp();
        }
        return;
    }

    // ---- consumers ----
    T w[C::KK];
#pragma unroll
    for (int q = 0; q < C::KK; ++q) w[q] = s_wt[q];
    const bool vec_ok = P.y_vec != 0;
    constexpr unsigned long long VMASK = (1ull << V) - 1ull;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // (Y may still be in use by the previous kernel)

    int it = 0;
    for (ItemIter I(P); I.img < P.batch; I.next(), ++it) {
        const int st = it % STAGES;
        const int img = I.img, tx = I.tx, ty = I.ty;
        const int xb = tx * TH + warp * V;  // this warp's first output row
        const int y0 = ty * C::TW;
        // (element staging: the producer warp's issue slots are the limit, so
        // the consumers sleep between polls instead of spinning beside it)
        if (P.notma)
            mbar_wait_backoff(&full[st], (uint32_t)((it / STAGES) & 1));
        else
            mbar_wait(&full[st], (uint32_t)((it / STAGES) & 1));
        // This warp's rows must all lie in verified segments (and the taps be
        // finite and non-zero) for the blocked path.
        const bool fast = FUSED || (P.fast_allowed && ((s_mask[st] >> (warp * V)) & VMASK) == VMASK);
        const T* xw = xs + (size_t)st * C::SF;
        T* ybase = reinterpret_cast<T*>(P.Y) + (long long)img * P.ldy;

        bool per_entry = !fast;
        if (fast) {
            T acc[V][CPT];
#pragma unroll
            for (int v = 0; v < V; ++v)
#pragma unroll
                for (int c = 0; c < CPT; ++c) acc[v][c] = (T)0;
            const T* xt = xw + (S * warp * V) * C::WC + S * CPT * lane;
#pragma unroll
            for (int jj = 0; jj < C::JJ; ++jj) {
                T xr[(C::VEC ? C::E : 1) * C::NV4];
#pragma unroll
                for (int q = 0; q < C::NV4; ++q) {
                    if constexpr (!C::VEC) {
                        xr[q] = xt[jj * C::WC + q];
                    } else if constexpr (F64) {
                        const double2 f = *reinterpret_cast<const double2*>(xt + jj * C::WC + 2 * q);
                        xr[2 * q] = f.x;
                        xr[2 * q + 1] = f.y;
                    } else {
                        const float4 f = *reinterpret_cast<const float4*>(xt + jj * C::WC + 4 * q);
                        xr[4 * q] = f.x;
                        xr[4 * q + 1] = f.y;
                        xr[4 * q + 2] = f.z;
                        xr[4 * q + 3] = f.w;
                    }
                }
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const int j = jj - S * v;
                    if (j >= 0 && j < K) {
#pragma unroll
                        for (int c = 0; c < CPT; ++c)
#pragma unroll
                            for (int ii = 0; ii < K; ++ii)
                                acc[v][c] = band_step(acc[v][c], w[j * K + ii], xr[DELTA + S * c + ii]);
                    }
                }
            }
            if (ZT) {
                T nf = (T)0;  // NaN iff some sum is not finite
#pragma unroll
                for (int v = 0; v < V; ++v)
#pragma unroll
                    for (int c = 0; c < CPT; ++c) nf = fma((T)0, acc[v][c], nf);
                per_entry = nf != (T)0;
            }
            const int ycol = y0 + CPT * lane;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int x = xb + v;
                if (per_entry || x >= P.mo) continue;
                T* yp = ybase + (long long)x * P.no + ycol;
                if constexpr (F64) {
                    if (vec_ok && ycol + CPT <= P.no) {
#pragma unroll
                        for (int c = 0; c + 1 < CPT; c += 2)
                            __stcs(reinterpret_cast<double2*>(yp + c), make_double2(acc[v][c], acc[v][c + 1]));
                    } else {
#pragma unroll
                        for (int c = 0; c < CPT; ++c)
                            if (ycol + c < P.no) __stcs(yp + c, acc[v][c]);
                    }
                } else if (vec_ok && ycol + CPT <= P.no) {
                    if (CPT == 4)
                        __stcs(reinterpret_cast<float4*>(yp),
                               make_float4(acc[v][0], acc[v][CPT > 1 ? 1 : 0], acc[v][CPT > 2 ? 2 : 0],
                                           acc[v][CPT > 3 ? 3 : 0]));
                    else
                        __stcs(reinterpret_cast<float2*>(yp), make_float2(acc[v][0], acc[v][CPT > 1 ? 1 : 0]));
                } else {
#pragma unroll
                    for (int c = 0; c < CPT; ++c)
                        if (ycol + c < P.no) __stcs(yp + c, acc[v][c]);
                }
            }
        }
        if (per_entry && P.csc) {
            // CSC storage (verified against these taps by the check): the
            // stored taps of each output in (j, i) = column-ascending order,
            // straight from the staged window.
            for (int v = 0; v < V; ++v) {
                const int x = xb + v;
                if (x >= P.mo) break;
                int jlo, jhi;
                tap_range_dev(x, P.m, K, S, P.p, jlo, jhi);
                for (int c = 0; c < CPT; ++c) {
                    const int y = y0 + CPT * lane + c;
                    if (y >= P.no) break;
                    int ilo, ihi;
                    tap_range_dev(y, P.n, K, S, P.p, ilo, ihi);
                    const T* xo = xw + (S * (x - tx * TH)) * C::WC + S * (y - y0) + DELTA;
                    T acc = (T)0;
                    for (int j = jlo; j < jhi; ++j)
                        for (int ii = ilo; ii < ihi; ++ii)
                            if (!ZT || ((P.nzmask >> (j * K + ii)) & 1ull))
                                acc = band_step(acc, s_wt[j * K + ii], xo[j * C::WC + ii]);
                    __stcs(ybase + (long long)x * P.no + y, acc);
                }
            }
        } else if (per_entry) {
            // Per-entry loop straight from the CSR (window-relative gathers).
            const int wr0 = S * tx * TH - P.p;
            const int wc0 = S * y0 - P.p - DELTA;
            for (int v = 0; v < V; ++v) {
                const int x = xb + v;
                if (x >= P.mo) break;
                for (int c = 0; c < CPT; ++c) {
                    const int y = y0 + CPT * lane + c;
                    if (y >= P.no) break;
                    const int r = x * P.no + y;
                    const int e1 = __ldg(P.row_ptr + r + 1);
                    T acc = (T)0;
                    for (int e = __ldg(P.row_ptr + r); e < e1; ++e) {
                        const int col = __ldg(P.col_idx + e);
                        if ((unsigned)col >= (unsigned)(P.m * P.n)) __trap();  // not a CSR of this shape
                        const int ri = col / P.n;
                        const int dr = ri - wr0, dc = col - ri * P.n - wc0;
                        // a column outside the staged window (a row that is not a conv
                        // row) is read from the image itself
                        const T xv = ((unsigned)dr < (unsigned)C::WR && (unsigned)dc < (unsigned)C::WC)
                                         ? xw[dr * C::WC + dc]
                                         : __ldg(reinterpret_cast<const T*>(P.X) + (long long)img * P.ldx + col);
                        // (fp64: the exact value when the handle keeps one)
                        const T v = F64 && P.vals64 ? (T)__ldg(P.vals64 + e) : (T)__ldg(P.vals + e);
                        acc = band_step(acc, v, xv);
                    }
                    __stcs(ybase + r, acc);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
}

// After a fused call: the rows of every segment whose check failed, for every
// image, recomputed from the CSR in stored order (per-entry, bit-exact).  A
// programmatic dependent of the fused kernel: resident early, it reads the
// flags only after griddepcontrol.wait (the fused grid complete and visible).
template <int TW>
__global__ void __launch_bounds__(256) conv_band_fixup(const BandParams P) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const long long nseg = (long long)P.mo * P.tiles_y;
    // one flag per thread; a chunk without failures costs one load and one barrier
    for (long long base = (long long)blockIdx.x * blockDim.x; base < nseg; base += (long long)gridDim.x * blockDim.x) {
        const long long mine = base + threadIdx.x;
        const bool bad = mine < nseg && P.seg_ok[mine] == 0;
        if (!__syncthreads_or(bad)) continue;
        for (long long seg = base; seg < min(nseg, base + (long long)blockDim.x); ++seg) {
            if (P.seg_ok[seg]) continue;  // block-uniform
            const int x = (int)(seg / P.tiles_y);
            const int y0 = (int)(seg - (long long)x * P.tiles_y) * TW;
            const int nr = min(TW, P.no - y0);
            const int r0 = x * P.no + y0;
            for (int q = threadIdx.x; q < nr * P.batch; q += blockDim.x) {
                const int img = q / nr, r = r0 + (q - img * nr);
                const float* X = P.X + (long long)img * P.ldx;
                float acc = 0.0f;
                for (int e = __ldg(P.row_ptr + r), e1 = __ldg(P.row_ptr + r + 1); e < e1; ++e)
                    acc = fmaf(__ldg(P.vals + e), __ldg(X + __ldg(P.col_idx + e)), acc);
                P.Y[(long long)img * P.ldy + r] = acc;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Host side: per-(k, s) blocking and launch.
// ---------------------------------------------------------------------------
namespace {

// The apply kernels (fused or not): a programmatic dependent of the previous
// kernel on the stream when bp.pdl (see conv_spmm_band's prologue).
template <typename Kern>
cudaError_t launch_band_kernel(Kern kern, unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                               const CUtensorMap* tmap, const BandParams& bp) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = bp.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, *tmap, bp);
}

template <typename Kern>
cudaError_t launch_pdl(Kern kern, unsigned grid, unsigned block, size_t smem, cudaStream_t st, const BandParams& bp) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, bp);
}

// Fused check + apply (conv_spmm_band<..., true>) and its fixup kernel.
template <int K, int S, int V, int CPT, int TH, int STAGES, int DELTA, bool ZT>
cudaError_t run_fused(const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, int sms) {
    using C = BandCfg<K, S, V, CPT, TH, STAGES, DELTA>;
    using FC = FusedCfg<K, S, V, CPT, TH, STAGES, DELTA>;
    constexpr size_t SMEM = FC::SMEM;
    if constexpr (FC::CHK == 0) {
        return cudaErrorNotSupported;
    } else {
        auto kern = conv_spmm_band<K, S, V, CPT, TH, STAGES, DELTA, true, ZT>;
        static std::atomic<int> occ[64];  // per device; 0 = not yet queried
        int dev = 0;
        cudaGetDevice(&dev);
        if (!occ[dev & 63]) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
            if (e != cudaSuccess) return e;
            int o = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, FC::THREADS, SMEM);
            if (e != cudaSuccess) return e;
            occ[dev & 63] = std::max(o, 1);
        }
        const long long items = (long long)bp.tiles * bp.batch;
        // every CTA also owns segments: at least one CTA per SM even for short batches
        const long long grid = std::min<long long>(std::max<long long>(items, sms), (long long)occ[dev & 63] * sms);
        cudaError_t e = launch_band_kernel(kern, (unsigned)grid, FC::THREADS, SMEM, st, tmap, bp);
        if (e != cudaSuccess) return e;
        if (!bp.fixup) return cudaSuccess;  // (failed segments raise the handle's verdict instead)
        const long long segs = (long long)bp.mo * bp.tiles_y;
        return launch_pdl(conv_band_fixup<C::TW>, (unsigned)std::min<long long>((segs + 255) / 256, sms), 256, 0, st,
                          bp);
    }
}

template <int K, int S, int V, int CPT, int TH, int STAGES, int DELTA, bool ZT = false>
cudaError_t run_cfg(const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, BandShape* shape,
                    int sms) {
    using C = BandCfg<K, S, V, CPT, TH, STAGES, DELTA>;
    static_assert(C::SMEM <= 227 * 1024, "band blocking exceeds shared memory");
    if (!shape && bp.fused) return run_fused<K, S, V, CPT, TH, STAGES, DELTA, ZT>(bp, tmap, st, sms);
    auto kern = conv_spmm_band<K, S, V, CPT, TH, STAGES, DELTA, false, ZT>;
    static std::atomic<int> occ[64];  // per device; 0 = not yet queried
    int dev = 0;
    cudaGetDevice(&dev);
    if (!occ[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e != cudaSuccess) return e;
        int o = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, C::THREADS, C::SMEM);
        if (e != cudaSuccess) return e;
        occ[dev & 63] = std::max(o, 1);
    }
    if (shape) {
        *shape = BandShape{TH, C::TW, C::WR, C::WC, (int)C::SMEM, C::THREADS, occ[dev & 63]};
        return cudaSuccess;
    }
    const long long items = (long long)bp.tiles * bp.batch;
    const long long grid = std::min<long long>(items, (long long)occ[dev & 63] * sms);
    return launch_band_kernel(kern, (unsigned)grid, C::THREADS, C::SMEM, st, tmap, bp);
}

template <int K, int S, int V, int CPT, int TH, int STAGES, bool ZT>
cudaError_t run_delta_z(int delta, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st,
                        BandShape* shape, int sms) {
    switch (delta) {
        case 0: return run_cfg<K, S, V, CPT, TH, STAGES, 0, ZT>(bp, tmap, st, shape, sms);
        case 1: return run_cfg<K, S, V, CPT, TH, STAGES, 1, ZT>(bp, tmap, st, shape, sms);
        case 2: return run_cfg<K, S, V, CPT, TH, STAGES, 2, ZT>(bp, tmap, st, shape, sms);
        default: return run_cfg<K, S, V, CPT, TH, STAGES, 3, ZT>(bp, tmap, st, shape, sms);
    }
}

// The default blocking of each (k, s); zero-tap transforms (bp.zt, only for
// launches -- the shape query is blocking-only) take the ZT instantiation.
// (zero-tap masks are 64 bits: k <= 7.  DELTA keeps every window's first
// column 16-byte aligned in global memory -- a TMA box may not start between
// 16-byte units -- also where the consumers read element by element, s = 3.)
template <int K, int S, int V, int CPT, int TH, int STAGES>
cudaError_t run_delta(int delta, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st,
                      BandShape* shape, int sms) {
    const bool zt = !shape && bp.zt;
    if constexpr (K * K > 64) {
        if (zt) return cudaErrorNotSupported;
        return run_delta_z<K, S, V, CPT, TH, STAGES, false>(delta, bp, tmap, st, shape, sms);
    } else {
        if (zt) return run_delta_z<K, S, V, CPT, TH, STAGES, true>(delta, bp, tmap, st, shape, sms);
        return run_delta_z<K, S, V, CPT, TH, STAGES, false>(delta, bp, tmap, st, shape, sms);
    }
}

// fp64 apply (two-kernel form only: the check runs first, as for fp32).
template <int K, int S, int V, int CPT, int TH, int STAGES, int DELTA, bool ZT>
cudaError_t run_cfg64(const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, BandShape* shape, int sms) {
    using C = BandCfg<K, S, V, CPT, TH, STAGES, DELTA, double>;
    static_assert(C::SMEM <= 227 * 1024, "fp64 blocking exceeds shared memory");
    auto kern = conv_spmm_band<K, S, V, CPT, TH, STAGES, DELTA, false, ZT, double>;
    static std::atomic<int> occ[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (!occ[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e != cudaSuccess) return e;
        int o = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, C::THREADS, C::SMEM);
        if (e != cudaSuccess) return e;
        occ[dev & 63] = std::max(o, 1);
    }
    if (shape) {
        *shape = BandShape{TH, C::TW, C::WR, C::WC, (int)C::SMEM, C::THREADS, occ[dev & 63]};
        return cudaSuccess;
    }
    const long long items = (long long)bp.tiles * bp.batch;
    const long long grid = std::min<long long>(items, (long long)occ[dev & 63] * sms);
    return launch_band_kernel(kern, (unsigned)grid, C::THREADS, C::SMEM, st, tmap, bp);
}

template <int K, int S, int V, int CPT, int TH, int STAGES>
cudaError_t run_delta64(int delta, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, BandShape* shape,
                        int sms) {
    const bool zt = !shape && bp.zt;
    if (delta == 0)
        return zt ? run_cfg64<K, S, V, CPT, TH, STAGES, 0, true>(bp, tmap, st, shape, sms)
                  : run_cfg64<K, S, V, CPT, TH, STAGES, 0, false>(bp, tmap, st, shape, sms);
    return zt ? run_cfg64<K, S, V, CPT, TH, STAGES, 1, true>(bp, tmap, st, shape, sms)
              : run_cfg64<K, S, V, CPT, TH, STAGES, 1, false>(bp, tmap, st, shape, sms);
}

template <int K, int S, int TW>
cudaError_t run_check(const BandParams& bp, cudaStream_t st, int sms) {
    (void)sms;
    using C = CheckCfg<K, S, TW>;
    using CS = CheckCfg<K, S, TW, csc_per<K, S, TW>(), S * TW>;  // (CSC staging)
    auto kern = bp.csc ? (bp.zt ? conv_band_check<K, S, TW, true, true> : conv_band_check<K, S, TW, false, true>)
                       : (bp.zt ? conv_band_check<K, S, TW, true, false> : conv_band_check<K, S, TW, false, false>);
    const int v = (bp.zt ? 1 : 0) + (bp.csc ? 2 : 0);
    static std::atomic<bool> init[4][64];
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t smem = bp.csc ? CS::SMEM : C::SMEM;
    const int warps = bp.csc ? CS::WARPS : C::WARPS;
    if (!init[v][dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        init[v][dev & 63] = true;
    }
    const long long segs = bp.csc ? (long long)bp.m * bp.tiles_b : (long long)bp.mo * bp.tiles_y;
    const long long grid = (segs + warps - 1) / warps;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(warps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = bp.pdl && opt(kOptPdl) != 2 ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, bp);
}

}  // namespace

}  // namespace spb
