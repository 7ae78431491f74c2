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
};

// ---------------------------------------------------------------------------
// 1. Band check: one warp per segment.
// ---------------------------------------------------------------------------
template <int K, int S, int TW>
__global__ void __launch_bounds__(256) conv_band_check(const BandParams P) {
    constexpr int KK = K * K;
    __shared__ uint32_t s_w[KK];
    for (int q = threadIdx.x; q < KK; q += blockDim.x) s_w[q] = __float_as_uint(__ldg(P.taps + q));
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const long long seg = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (seg >= (long long)P.mo * P.tiles_y) return;
    const int x = (int)(seg / P.tiles_y);
    const int ty = (int)(seg - (long long)x * P.tiles_y);
    const int y0 = ty * TW;
    const int nr = min(TW, P.no - y0);
    const int r0 = x * P.no + y0;

    int jlo, jhi;
    tap_range_dev(x, P.m, K, S, P.p, jlo, jhi);
    bool ok = true;
    bool full = (jlo == 0 && jhi == K);
    int a_first[TW / 32];
#pragma unroll
    for (int q = 0; q < TW / 32; ++q) {
        const int l = lane + 32 * q;
        a_first[q] = 0;
        if (l < nr) {
            int ilo, ihi;
            tap_range_dev(y0 + l, P.n, K, S, P.p, ilo, ihi);
            const int a = __ldg(P.row_ptr + r0 + l), b = __ldg(P.row_ptr + r0 + l + 1);
            ok &= (b - a) == (jhi - jlo) * (ihi - ilo);
            full &= (ilo == 0 && ihi == K);
            a_first[q] = a;
        }
    }
    full = __all_sync(0xffffffffu, full);
    if (full && __all_sync(0xffffffffu, ok)) {
        // Contiguous run of nr*KK pairs starting at row_ptr[r0].
        const int S0 = __shfl_sync(0xffffffffu, a_first[0], 0);
#pragma unroll
        for (int q = 0; q < TW / 32; ++q) {
            const int l = lane + 32 * q;
            if (l < nr) ok &= a_first[q] == S0 + l * KK;
        }
        const int base = (S * x - P.p) * P.n + (S * y0 - P.p);
        const int len = nr * KK;
        const int32_t* cp = P.col_idx + S0;
        const float* vp = P.vals + S0;
        uint32_t bad = 0;
        constexpr int U = 8;
        for (int d0 = 0; d0 < len; d0 += 32 * U) {
            int c[U];
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int d = d0 + lane + 32 * u;
                c[u] = d < len ? __ldg(cp + d) : 0;
                v[u] = d < len ? __float_as_uint(__ldg(vp + d)) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int d = d0 + lane + 32 * u;
                if (d < len) {
                    const int l = d / KK, q = d - l * KK;
                    const int j = q / K, i = q - j * K;
                    bad |= (uint32_t)(c[u] - (base + S * l + j * P.n + i)) | (v[u] ^ s_w[q]);
                }
            }
        }
        ok &= bad == 0u;
    } else {
        // Border segment: each lane walks its own rows.
#pragma unroll
        for (int q = 0; q < TW / 32; ++q) {
            const int l = lane + 32 * q;
            if (l < nr && ok) {
                const int y = y0 + l;
                int ilo, ihi;
                tap_range_dev(y, P.n, K, S, P.p, ilo, ihi);
                int e = a_first[q];
                for (int j = jlo; j < jhi; ++j) {
                    const int rowc = (S * x + j - P.p) * P.n + (S * y - P.p);
                    for (int i = ilo; i < ihi; ++i, ++e)
                        ok &= (__ldg(P.col_idx + e) == rowc + i) &&
                              (__float_as_uint(__ldg(P.vals + e)) == s_w[j * K + i]);
                }
            }
        }
    }
    ok = __all_sync(0xffffffffu, ok);
    if (lane == 0) P.seg_ok[seg] = ok ? 1 : 0;
}

// ---------------------------------------------------------------------------
// 2. Register-blocked apply.
// ---------------------------------------------------------------------------
template <int K, int S, int V, int CPT, int TH, int STAGES, int DELTA>
__global__ void __launch_bounds__(BandCfg<K, S, V, CPT, TH, STAGES, DELTA>::THREADS, 1)
    conv_spmm_band(const __grid_constant__ CUtensorMap tmap, const BandParams P) {
    using C = BandCfg<K, S, V, CPT, TH, STAGES, DELTA>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + STAGES;
    float* xs = reinterpret_cast<float*>(smem + 128);

    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const long long items = (long long)P.tiles * P.batch;  // item = img * tiles + tile

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
        // ---- producer: one elected lane issues the window loads ----
        if (lane == 0) {
            int it = 0;
            for (long long i = blockIdx.x; i < items; i += gridDim.x, ++it) {
                const int st = it % STAGES;
                if (it >= STAGES) mbar_wait(&empty[st], (uint32_t)(((it / STAGES) - 1) & 1));
                const int img = (int)(i / P.tiles);
                const int tile = (int)(i - (long long)img * P.tiles);
                const int tx = tile / P.tiles_y, ty = tile - tx * P.tiles_y;
                const int wr0 = S * tx * TH - P.p;
                const int wc0 = S * ty * C::TW - P.p - DELTA;
                mbar_expect_tx(&full[st], (uint32_t)(C::WIN * 4));
                tma_load_3d(xs + (size_t)st * C::SF, &tmap, wc0, wr0, img, &full[st]);
            }
        }
        return;
    }

    // ---- consumers ----
    float w[C::KK];
#pragma unroll
    for (int q = 0; q < C::KK; ++q) w[q] = __ldg(P.taps + q);
    const bool vec_ok = P.y_vec != 0;

    int it = 0;
    for (long long i = blockIdx.x; i < items; i += gridDim.x, ++it) {
        const int st = it % STAGES;
        const int img = (int)(i / P.tiles);
        const int tile = (int)(i - (long long)img * P.tiles);
        const int tx = tile / P.tiles_y, ty = tile - tx * P.tiles_y;
        const int xb = tx * TH + warp * V;  // this warp's first output row
        const int y0 = ty * C::TW;
        // This warp's rows must all lie in verified segments.
        bool ok = true;
        if (lane < V) {
            const int x = xb + lane;
            ok = x >= P.mo || P.seg_ok[(long long)x * P.tiles_y + ty] != 0;
        }
        const bool fast = __all_sync(0xffffffffu, ok) && P.fast_allowed;

        mbar_wait(&full[st], (uint32_t)((it / STAGES) & 1));
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
cudaError_t run_check(const BandParams& bp, cudaStream_t st) {
    const long long segs = (long long)bp.mo * bp.tiles_y;
    const long long grid = (segs + 7) / 8;
    conv_band_check<K, S, TW><<<(unsigned)grid, 256, 0, st>>>(bp);
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
    if (k == 3 && s == 1) return run_delta<3, 1, 4, 4, 32, 4>(delta, bp, tmap, st, shape, sms);
    if (k == 5 && s == 1) return run_delta<5, 1, 4, 4, 32, 4>(delta, bp, tmap, st, shape, sms);
    if (k == 3 && s == 2) return run_delta<3, 2, 4, 2, 16, 4>(delta, bp, tmap, st, shape, sms);
    if (k == 5 && s == 2) return run_delta<5, 2, 4, 2, 16, 4>(delta, bp, tmap, st, shape, sms);
    if (k == 7 && s == 2) return run_delta<7, 2, 4, 2, 16, 4>(delta, bp, tmap, st, shape, sms);
    return cudaErrorInvalidValue;
}

cudaError_t launch_band_check(int k, int s, const BandParams& bp, cudaStream_t st) {
    if (k == 3 && s == 1) return run_check<3, 1, 128>(bp, st);
    if (k == 5 && s == 1) return run_check<5, 1, 128>(bp, st);
    if (k == 3 && s == 2) return run_check<3, 2, 64>(bp, st);
    if (k == 5 && s == 2) return run_check<5, 2, 64>(bp, st);
    if (k == 7 && s == 2) return run_check<7, 2, 64>(bp, st);
    return cudaErrorInvalidValue;
}

}  // namespace spb
