// spmm_band.cu -- the hot path: SpMM of the conv transform T against an
// image-major batch, as two kernels per call.
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
//    An interior segment (every row full) is one contiguous run of TW*k*k
//    (col, val) pairs: a warp streams it with coalesced loads and compares
//    against the closed-form pattern.  Border segments are walked row by row.
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
//    Blocked == per-entry, bit for bit: a tap that lands in the zero padding
//    executes fmaf(w, +0.0f, acc), which returns acc unchanged (acc starts at
//    +0 and is never -0 under round-to-nearest, w is finite), so executing or
//    skipping the clipped taps is indistinguishable, and every output still
//    sees its stored taps in (j, i) = column-ascending order.
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
constexpr int cmax(int a, int b) { return a > b ? a : b; }

}  // namespace

// ---------------------------------------------------------------------------
// Geometry of one instantiation.
// ---------------------------------------------------------------------------
template <int K, int S, int V, int CPT, int TH, int STAGES, int DELTA>
struct BandCfg {
    static_assert(S * CPT == 4, "thread columns must start 16-byte aligned in the window");
    static_assert(TH % V == 0, "TH must be a multiple of V");
    static constexpr int KK = K * K;
    static constexpr int TW = 32 * CPT;                 // output columns per tile
    static constexpr int NX = S * (CPT - 1) + K;        // window columns one thread reads per row
    static constexpr int NV4 = (DELTA + NX + 3) / 4;    // float4 loads per row
    static constexpr int JJ = S * (V - 1) + K;          // window rows one thread reads
    static constexpr int WR = S * (TH - 1) + K;         // window rows
    static constexpr int WC = cmax(round_up(S * (TW - 1) + K + DELTA, 4), 4 * 31 + 4 * NV4);
    static constexpr int WIN = WR * WC;
    static constexpr int CWARPS = TH / V;               // consumer warps
    static constexpr int THREADS = 32 * (CWARPS + 1);   // + one producer warp
    static constexpr int SF = round_up(WIN, 32);        // floats per stage (128-byte aligned)
    static constexpr size_t SMEM = 128 + (size_t)STAGES * SF * 4;
    static_assert(WC <= 256 && WR <= 256, "TMA box limit");
    static_assert(TH <= 32, "one producer lane per tile row");
    static_assert(STAGES * 20 <= 128, "barriers + flag masks fit the 128-byte header");
};

// ---------------------------------------------------------------------------
// 1. Band check: one warp per segment.
// ---------------------------------------------------------------------------
template <int K, int S, int TW>
struct CheckCfg {
    static constexpr int KK = K * K;
    static constexpr int RUN = TW * KK;                    // entries of an interior segment
    static constexpr int BUFW = (RUN + 3 + 3) / 4 * 4;     // 16-byte aligned superset
    static constexpr size_t WARP_BYTES = 2ull * 2 * BUFW * 4;  // 2 buffers x (cols + vals)
    static constexpr int WARPS = (int)(200 * 1024 / WARP_BYTES) < 8 ? (int)(200 * 1024 / WARP_BYTES) : 8;
    static constexpr size_t SMEM = 128 + (size_t)WARPS * WARP_BYTES;
    static_assert(WARPS >= 1, "segment too large for shared memory");
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <int K, int S, int TW>
__global__ void __launch_bounds__(CheckCfg<K, S, TW>::WARPS * 32, 1) conv_band_check(const BandParams P) {
    using C = CheckCfg<K, S, TW>;
    constexpr int KK = K * K;
    constexpr int RPL = TW / 32;  // rows per lane
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + 2 * warp;
    int* buf = reinterpret_cast<int*>(smem + 128 + (size_t)warp * C::WARP_BYTES);
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_fence_init();
    }
    __syncwarp();
    __shared__ uint32_t s_w[KK];  // taps for the border walk (runtime-indexed)
    for (int q = threadIdx.x; q < KK; q += blockDim.x) s_w[q] = __float_as_uint(__ldg(P.taps + q));
    __syncthreads();
    uint32_t w[KK];  // taps for the interior check (compile-time indexed)
#pragma unroll
    for (int q = 0; q < KK; ++q) w[q] = s_w[q];

    // Each warp owns a contiguous range of segments (consecutive memory, and
    // every warp meets its share of border segments).
    const long long nseg_all = (long long)P.mo * P.tiles_y;
    const long long nw = (long long)gridDim.x * C::WARPS;
    const long long gw = (long long)blockIdx.x * C::WARPS + warp;
    const long long seg_lo = nseg_all * gw / nw, nseg = nseg_all * (gw + 1) / nw;
    const long long stride = 1;

    // Segment geometry + closed-form start (dense taps): rows before (x, y0)
    // = CX(x) * SY + cx(x) * CY(y0)  (Theorem 2.1 prefix sums).
    struct Seg {
        int x, y0, nr, r0, jlo, jhi, S0;
        bool full;
    };
    auto geom = [&](long long seg) {
        Seg g;
        g.x = (int)(seg / P.tiles_y);
        const int ty = (int)(seg - (long long)g.x * P.tiles_y);
        g.y0 = ty * TW;
        g.nr = min(TW, P.no - g.y0);
        g.r0 = g.x * P.no + g.y0;
        tap_range_dev(g.x, P.m, K, S, P.p, g.jlo, g.jhi);
        int cxb = 0, cyb = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            cxb += slides_before(g.x, j, P.m, S, P.p);
            cyb += slides_before(g.y0, j, P.n, S, P.p);
        }
        g.S0 = cxb * P.sy + (g.jhi - g.jlo) * cyb;
        // interior: every row of the segment stores all K*K taps
        const int ylast = g.y0 + g.nr - 1;
        g.full = g.jlo == 0 && g.jhi == K && S * g.y0 - P.p >= 0 && S * ylast - P.p + K <= P.n &&
                 (long long)g.S0 + g.nr * KK <= (long long)P.nnz;  // (zero taps: prediction past the end)
        return g;
    };
    auto issue = [&](const Seg& g, int b) {  // lane 0: bulk-copy the run into buffer b
        const int abase = g.S0 & ~3;
        const uint32_t bytes = (uint32_t)(((g.S0 + g.nr * KK - abase + 3) & ~3) * 4);
        int* dst = buf + b * 2 * C::BUFW;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bars[b], 2 * bytes);
        bulk_g2s(dst, P.col_idx + abase, bytes, &bars[b]);
        bulk_g2s(dst + C::BUFW, P.vals + abase, bytes, &bars[b]);
    };

    long long seg = seg_lo;
    if (seg >= nseg) return;
    Seg cur = geom(seg);
    if (cur.full && lane == 0) issue(cur, 0);
    uint32_t phases = 0u;  // bit b: parity of buffer b's next completion
    for (int i = 0; seg < nseg; ++i, seg += stride) {
        const int b = i & 1;
        // row_ptr of this segment (nr + 1 values)
        int a_row[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            const int l = lane + 32 * q;
            a_row[q] = l < cur.nr ? __ldg(P.row_ptr + cur.r0 + l) : 0;
        }
        const int a_end = __ldg(P.row_ptr + cur.r0 + cur.nr);
        // prefetch the next segment's run into the other buffer
        Seg nxt{};
        const bool has_next = seg + stride < nseg;
        if (has_next) {
            nxt = geom(seg + stride);
            __syncwarp();  // this warp finished reading buffer b^1 (segment i-1)
            if (nxt.full && lane == 0) issue(nxt, b ^ 1);
        }
        bool ok = true;
        if (cur.full) {
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int l = lane + 32 * q;
                if (l < cur.nr) ok &= a_row[q] == cur.S0 + l * KK;
            }
            ok &= a_end == cur.S0 + cur.nr * KK;
            mbar_wait(&bars[b], (phases >> b) & 1u);
            phases ^= 1u << b;
            const int* cb = buf + b * 2 * C::BUFW + (cur.S0 & 3);
            const uint32_t* vb = reinterpret_cast<const uint32_t*>(cb + C::BUFW);
            uint32_t bad = 0;
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int l = lane + 32 * q;
                if (l < cur.nr) {
                    const int rb = (S * cur.x - P.p) * P.n + S * (cur.y0 + l) - P.p;
                    const int* cl = cb + l * KK;
                    const uint32_t* vl = vb + l * KK;
#pragma unroll
                    for (int j = 0; j < K; ++j)
#pragma unroll
                        for (int ii = 0; ii < K; ++ii)
                            bad |= (uint32_t)(cl[j * K + ii] - (rb + j * P.n + ii)) | (vl[j * K + ii] ^ w[j * K + ii]);
                }
            }
            ok &= bad == 0u;
        } else {
            // Border segment: each lane walks its own rows from global memory,
            // every (col, val) load of a row in flight at once.
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int l = lane + 32 * q;
                if (l < cur.nr) {
                    const int y = cur.y0 + l;
                    int ilo, ihi;
                    tap_range_dev(y, P.n, K, S, P.p, ilo, ihi);
                    const int bnd = __ldg(P.row_ptr + cur.r0 + l + 1);
                    if (bnd - a_row[q] != (cur.jhi - cur.jlo) * (ihi - ilo)) {
                        ok = false;
                        continue;
                    }
                    const int rb = (S * cur.x - P.p) * P.n + (S * y - P.p);
                    int e = a_row[q];
                    uint32_t bad = 0;
#pragma unroll
                    for (int j = 0; j < K; ++j)
#pragma unroll
                        for (int ii = 0; ii < K; ++ii)
                            if (j >= cur.jlo && j < cur.jhi && ii >= ilo && ii < ihi) {
                                bad |= (uint32_t)(__ldg(P.col_idx + e) - (rb + j * P.n + ii)) |
                                       (__float_as_uint(__ldg(P.vals + e)) ^ w[j * K + ii]);
                                ++e;
                            }
                    ok &= bad == 0u;
                }
            }
        }
        ok = __all_sync(0xffffffffu, ok);
        if (lane == 0) P.seg_ok[seg] = ok ? 1 : 0;
        cur = nxt;
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
template <int K, int S, int V, int CPT, int TH, int STAGES, int DELTA>
__global__ void __launch_bounds__(BandCfg<K, S, V, CPT, TH, STAGES, DELTA>::THREADS, 1)
    conv_spmm_band(const __grid_constant__ CUtensorMap tmap, const BandParams P) {
    using C = BandCfg<K, S, V, CPT, TH, STAGES, DELTA>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + STAGES;
    unsigned* s_mask = reinterpret_cast<unsigned*>(empty + STAGES);  // per-stage row flags
    float* xs = reinterpret_cast<float*>(smem + 128);

    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;

    if (t == 0) {
        tma_prefetch_desc(&tmap);
        for (int st = 0; st < STAGES; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], C::CWARPS);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == C::CWARPS) {
        // ---- producer warp: per item, the tile rows' band-check flags (one
        // lane per row, folded into a per-stage bit mask) and the window load
        // (one elected lane).  Running STAGES items ahead hides the flag
        // loads' latency from the consumers.
        int it = 0;
        for (ItemIter I(P); I.img < P.batch; I.next(), ++it) {
            const int st = it % STAGES;
            bool f = true;
            if (lane < TH) {
                const int x = I.tx * TH + lane;
                f = x >= P.mo || __ldg(P.seg_ok + (long long)x * P.tiles_y + I.ty) != 0;
            }
            const unsigned rows_ok = __ballot_sync(0xffffffffu, f);
            if (lane == 0) {
                if (it >= STAGES) mbar_wait(&empty[st], (uint32_t)(((it / STAGES) - 1) & 1));
                s_mask[st] = rows_ok;
                const int wr0 = S * I.tx * TH - P.p;
                const int wc0 = S * I.ty * C::TW - P.p - DELTA;
                mbar_expect_tx(&full[st], (uint32_t)(C::WIN * 4));
                tma_load_3d(xs + (size_t)st * C::SF, &tmap, wc0, wr0, I.img, &full[st]);
            }
            __syncwarp();
        }
        return;
    }

    // ---- consumers ----
    float w[C::KK];
#pragma unroll
    for (int q = 0; q < C::KK; ++q) w[q] = __ldg(P.taps + q);
    const bool vec_ok = P.y_vec != 0;
    constexpr unsigned VMASK = (1u << V) - 1u;

    int it = 0;
    for (ItemIter I(P); I.img < P.batch; I.next(), ++it) {
        const int st = it % STAGES;
        const int img = I.img, tx = I.tx, ty = I.ty;
        const int xb = tx * TH + warp * V;  // this warp's first output row
        const int y0 = ty * C::TW;
        mbar_wait(&full[st], (uint32_t)((it / STAGES) & 1));
        // This warp's rows must all lie in verified segments (and the taps be
        // finite and non-zero) for the blocked path.
        const bool fast = P.fast_allowed && ((s_mask[st] >> (warp * V)) & VMASK) == VMASK;
        const float* xw = xs + (size_t)st * C::SF;
        float* ybase = P.Y + (long long)img * P.ldy;

        if (fast) {
            float acc[V][CPT];
#pragma unroll
            for (int v = 0; v < V; ++v)
#pragma unroll
                for (int c = 0; c < CPT; ++c) acc[v][c] = 0.0f;
            const float* xt = xw + (S * warp * V) * C::WC + 4 * lane;
#pragma unroll
            for (int jj = 0; jj < C::JJ; ++jj) {
                float xr[4 * C::NV4];
#pragma unroll
                for (int q = 0; q < C::NV4; ++q) {
                    const float4 f = *reinterpret_cast<const float4*>(xt + jj * C::WC + 4 * q);
                    xr[4 * q] = f.x;
                    xr[4 * q + 1] = f.y;
                    xr[4 * q + 2] = f.z;
                    xr[4 * q + 3] = f.w;
                }
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const int j = jj - S * v;
                    if (j >= 0 && j < K) {
#pragma unroll
                        for (int c = 0; c < CPT; ++c)
#pragma unroll
                            for (int ii = 0; ii < K; ++ii)
                                acc[v][c] = fmaf(w[j * K + ii], xr[DELTA + S * c + ii], acc[v][c]);
                    }
                }
            }
            const int ycol = y0 + CPT * lane;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int x = xb + v;
                if (x >= P.mo) continue;
                float* yp = ybase + (long long)x * P.no + ycol;
                if (vec_ok && ycol + CPT <= P.no) {
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
        } else {
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
                    float acc = 0.0f;
                    for (int e = __ldg(P.row_ptr + r); e < e1; ++e) {
                        const int col = __ldg(P.col_idx + e);
                        const int ri = col / P.n;
                        const int dr = ri - wr0, dc = col - ri * P.n - wc0;
                        if ((unsigned)dr >= (unsigned)C::WR || (unsigned)dc >= (unsigned)C::WC) __trap();
                        acc = fmaf(__ldg(P.vals + e), xw[dr * C::WC + dc], acc);
                    }
                    __stcs(ybase + r, acc);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
}

// ---------------------------------------------------------------------------
// Host side: per-(k, s) blocking and launch.
// ---------------------------------------------------------------------------
namespace {

template <int K, int S, int V, int CPT, int TH, int STAGES, int DELTA>
cudaError_t run_cfg(const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st, BandShape* shape,
                    int sms) {
    using C = BandCfg<K, S, V, CPT, TH, STAGES, DELTA>;
    auto kern = conv_spmm_band<K, S, V, CPT, TH, STAGES, DELTA>;
    static int occ[64] = {};
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
    kern<<<(unsigned)grid, C::THREADS, C::SMEM, st>>>(*tmap, bp);
    return cudaGetLastError();
}

template <int K, int S, int V, int CPT, int TH, int STAGES>
cudaError_t run_delta(int delta, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st,
                      BandShape* shape, int sms) {
    switch (delta) {
        case 0: return run_cfg<K, S, V, CPT, TH, STAGES, 0>(bp, tmap, st, shape, sms);
        case 1: return run_cfg<K, S, V, CPT, TH, STAGES, 1>(bp, tmap, st, shape, sms);
        case 2: return run_cfg<K, S, V, CPT, TH, STAGES, 2>(bp, tmap, st, shape, sms);
        default: return run_cfg<K, S, V, CPT, TH, STAGES, 3>(bp, tmap, st, shape, sms);
    }
}

template <int K, int S, int TW>
cudaError_t run_check(const BandParams& bp, cudaStream_t st, int sms) {
    using C = CheckCfg<K, S, TW>;
    auto kern = conv_band_check<K, S, TW>;
    static int occ[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!occ[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e != cudaSuccess) return e;
        int o = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, C::WARPS * 32, C::SMEM);
        if (e != cudaSuccess) return e;
        occ[dev & 63] = std::max(o, 1);
    }
    const long long segs = (long long)bp.mo * bp.tiles_y;
    const long long want = (segs + C::WARPS - 1) / C::WARPS;
    const long long grid = std::min<long long>(want, (long long)occ[dev & 63] * sms);
    kern<<<(unsigned)grid, C::WARPS * 32, C::SMEM, st>>>(bp);
    return cudaGetLastError();
}

}  // namespace

bool band_supported(int k, int s) {
    return (s == 1 && (k == 3 || k == 5)) || (s == 2 && (k == 3 || k == 5 || k == 7));
}

int band_tile_width(int k, int s) {
    (void)k;
    return s == 1 ? 128 : 64;
}

// delta = (box start alignment shift) = (S*y0 - p) mod 4 with y0 a multiple
// of the tile width: uniform over the launch.
cudaError_t launch_band(int k, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st,
                        BandShape* shape, int sms) {
    const int delta = ((-bp.p) % 4 + 4) % 4;
    // Blocking variants for tuning experiments (SPCONV_B200_VARIANT; 0 = default),
    // instantiated only for the alignment shift of the benchmark configs.
    static const int var = std::getenv("SPCONV_B200_VARIANT") ? std::atoi(std::getenv("SPCONV_B200_VARIANT")) : 0;
    if (k == 3 && s == 1) {
        if (delta == 3 && var == 1) return run_cfg<3, 1, 4, 4, 16, 4, 3>(bp, tmap, st, shape, sms);
        if (delta == 3 && var == 2) return run_cfg<3, 1, 8, 4, 32, 4, 3>(bp, tmap, st, shape, sms);
        if (delta == 3 && var == 3) return run_cfg<3, 1, 4, 4, 32, 3, 3>(bp, tmap, st, shape, sms);
        if (delta == 3 && var == 4) return run_cfg<3, 1, 2, 4, 16, 4, 3>(bp, tmap, st, shape, sms);
        return run_delta<3, 1, 4, 4, 32, 4>(delta, bp, tmap, st, shape, sms);
    }
    if (k == 5 && s == 1) return run_delta<5, 1, 4, 4, 32, 4>(delta, bp, tmap, st, shape, sms);
    if (k == 3 && s == 2) return run_delta<3, 2, 4, 2, 16, 4>(delta, bp, tmap, st, shape, sms);
    if (k == 5 && s == 2) return run_delta<5, 2, 4, 2, 16, 4>(delta, bp, tmap, st, shape, sms);
    if (k == 7 && s == 2) {
        if (delta == 1 && var == 1) return run_cfg<7, 2, 4, 2, 16, 3, 1>(bp, tmap, st, shape, sms);
        if (delta == 1 && var == 2) return run_cfg<7, 2, 2, 2, 16, 3, 1>(bp, tmap, st, shape, sms);
        if (delta == 1 && var == 3) return run_cfg<7, 2, 4, 2, 32, 2, 1>(bp, tmap, st, shape, sms);
        if (delta == 1 && var == 4) return run_cfg<7, 2, 2, 2, 8, 4, 1>(bp, tmap, st, shape, sms);
        return run_delta<7, 2, 4, 2, 16, 4>(delta, bp, tmap, st, shape, sms);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_band_check(int k, int s, const BandParams& bp, cudaStream_t st, int sms) {
    if (k == 3 && s == 1) return run_check<3, 1, 128>(bp, st, sms);
    if (k == 5 && s == 1) return run_check<5, 1, 128>(bp, st, sms);
    if (k == 3 && s == 2) return run_check<3, 2, 64>(bp, st, sms);
    if (k == 5 && s == 2) return run_check<5, 2, 64>(bp, st, sms);
    if (k == 7 && s == 2) return run_check<7, 2, 64>(bp, st, sms);
    return cudaErrorInvalidValue;
}

}  // namespace spb
