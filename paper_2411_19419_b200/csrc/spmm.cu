// spmm.cu -- SpMV / SpMM of T against image-major batches: the general kernels.
//
// Replaces spmv + detail::spmv_csr_rows (inc/sparse.hpp:180-192, 214-261) and
// the per-image convolve loop of its callers (inc/conv.hpp:207-215,
// inc/bench.hpp:240-248).  Accumulation contract of every kernel:
//     acc = +0.0f; for e in row (column-ascending): acc = fmaf(val[e], x[col[e]], acc)
// i.e. the reference's sequential row loop in fp32 with one rounding per step.
//
// conv_spmm_tiled -- any transform built by csr_build (any k, s, p, zero or
//   non-finite taps).  A CTA owns a TH x 32 block of output pixels (TH*32 rows
//   of T; warp = one image row of the block, lane = one output column).
//   Prologue: each thread reads its row's (col, val) pairs from the CSR once and
//   rewrites every column as an offset into the CTA's input window (the
//   (TH-1)s+k x 31s+k patch every entry of the block falls in); the pairs live
//   tap-major in shared memory ([q][thread], bank-conflict free).  Main loop:
//   the windows of BT images at a time are staged into shared memory by ONE
//   TMA 3-D box load (cols x rows x images; out-of-range coordinates
//   zero-fill), multi-buffered on mbarriers; each thread accumulates its row
//   for BT images.  The register-blocked fast path for the common geometries is
//   conv_band_check + conv_spmm_band (spmm_band.cu).
// csr_spmm_generic -- any CSR (uploaded host matrices): thread per (row,
//   image), x gathered through L1.
// csr_spmv_bulk -- the latency kernel for batch <= 2 (below).
// csr_spmv_unrolled -- thread per row, a cross-check path (SPCONV_B200_PATH=spmv_plain).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.h"
#include "tma.cuh"

namespace spb {

namespace {
constexpr int kTileW = 32;
inline __host__ __device__ int stage_floats(int bt, int win) { return (bt * win + 31) & ~31; }
}  // namespace

size_t tiled_smem_bytes(int th, int wr, int wc, int k2max, int bt, int stages) {
    const size_t bars = 128;  // mbarriers, padded so the windows stay 128B-aligned
    const size_t win = (size_t)stages * stage_floats(bt, wr * wc) * sizeof(float);
    const size_t pairs = (size_t)k2max * th * kTileW * 8;
    return bars + win + pairs;
}

template <int BT>
__global__ void __launch_bounds__(256) conv_spmm_tiled(const __grid_constant__ CUtensorMap tmap,
                                                       const TiledParams P) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int TILE = P.th * kTileW;
    const int t = threadIdx.x;
    const int win = P.wr * P.wc;
    const int stages = P.use_tma ? P.stages : 1;
    const int sf = stage_floats(BT, win);

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    float* xs = reinterpret_cast<float*>(smem + 128);
    int32_t* s_off = reinterpret_cast<int32_t*>(xs + (size_t)stages * sf);
    float* s_val = reinterpret_cast<float*>(s_off + P.k2max * TILE);

    const int tx = blockIdx.x / P.tiles_y, ty = blockIdx.x - tx * P.tiles_y;
    const int x0 = tx * P.th, y0 = ty * kTileW;
    const int x = x0 + (t >> 5), y = y0 + (t & 31);
    const bool valid = x < P.mo && y < P.no;
    const int r = x * P.no + y;
    const int wr0 = P.s * x0 - P.p;
    const int wc0 = (P.s * y0 - P.p) & ~3;  // floor to a 16B-aligned column

    const int G = (P.batch + BT - 1) / BT;

    // Kick off the first window loads before touching the CSR.
    if (P.use_tma && t == 0) {
        tma_prefetch_desc(&tmap);
        for (int st = 0; st < stages; ++st) mbar_init(&bars[st], 1);
        mbar_fence_init();
        const uint32_t bytes = (uint32_t)(BT * win * sizeof(float));
        for (int st = 0; st < stages && st < G; ++st) {
            mbar_expect_tx(&bars[st], bytes);
            tma_load_3d(xs + (size_t)st * sf, &tmap, wc0, wr0, st * BT, &bars[st]);
        }
    }

    // Prologue: this row's CSR entries -> window offsets, tap-major in smem.
    int cnt = 0;
    if (valid) {
        const int e0 = __ldg(P.row_ptr + r);
        cnt = __ldg(P.row_ptr + r + 1) - e0;
        bool bad = cnt > P.k2max;
        cnt = bad ? 0 : cnt;
#pragma unroll 4
        for (int q = 0; q < cnt; ++q) {
            const int c = __ldg(P.col_idx + e0 + q);
            const float v = __ldg(P.vals + e0 + q);
            const int ri = c / P.n;
            const int dr = ri - wr0, dc = c - ri * P.n - wc0;
            bad |= (unsigned)dr >= (unsigned)P.wr || (unsigned)dc >= (unsigned)P.wc;
            s_off[q * TILE + t] = dr * P.wc + dc;
            s_val[q * TILE + t] = v;
        }
        if (bad) __trap();  // entry outside the tile window: not a transform of this geometry
    }
    __syncthreads();  // mbarrier init visible to all waiters

    for (int g = 0; g < G; ++g) {
        const int st = g % stages;
        float* xw = xs + (size_t)st * sf;
        if (P.use_tma) {
            mbar_wait(&bars[st], (uint32_t)((g / stages) & 1));
        } else {
            // Cooperative staging for geometries TMA cannot describe
            // (row pitch not a multiple of 16 bytes, window > 256).
            for (int idx = t; idx < BT * win; idx += blockDim.x) {
                const int b = idx / win, rem = idx - b * win;
                const int rr = rem / P.wc, cc = rem - rr * P.wc;
                const int gr = wr0 + rr, gc = wc0 + cc, img = g * BT + b;
                float v = 0.0f;
                if (gr >= 0 && gr < P.m && gc >= 0 && gc < P.n && img < P.batch)
                    v = __ldg(P.X + (int64_t)img * P.ldx + (int64_t)gr * P.n + gc);
                xw[idx] = v;
            }
            __syncthreads();
        }

        float acc[BT];
#pragma unroll
        for (int b = 0; b < BT; ++b) acc[b] = 0.0f;
#pragma unroll 3
        for (int q = 0; q < cnt; ++q) {
            const float* xq = xw + s_off[q * TILE + t];
            const float v = s_val[q * TILE + t];
#pragma unroll
            for (int b = 0; b < BT; ++b) acc[b] = fmaf(v, xq[b * win], acc[b]);
        }
        if (valid) {
#pragma unroll
            for (int b = 0; b < BT; ++b) {
                const int img = g * BT + b;
                if (img < P.batch) __stcs(P.Y + (int64_t)img * P.ldy + r, acc[b]);
            }
        }
        __syncthreads();  // every thread is done reading stage st
        if (P.use_tma && t == 0 && g + stages < G) {
            mbar_expect_tx(&bars[st], (uint32_t)(BT * win * sizeof(float)));
            tma_load_3d(xw, &tmap, wc0, wr0, (g + stages) * BT, &bars[st]);
        }
    }
}

// (chunk > 0: columns cut into chunks of `chunk`, one partial per chunk added
// to y in chunk order -- the reference's CSC thread combine with nt threads.)
// fp64 SpMM with the reference's own arithmetic: per row acc = 0.0; for each
// stored entry in order acc = acc + (double)val * x (one rounded multiply, one
// rounded add -- no contraction, as the reference's Release build evaluates
// inc/sparse.hpp:185-191).  With fp32-representable taps the stored values are
// the reference's exactly, so the output is bit-identical to its spmv().
__global__ void __launch_bounds__(256) csr_spmm_f64(const F64Params P) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= P.rows) return;
    const int e0 = __ldg(P.row_ptr + r), e1 = __ldg(P.row_ptr + r + 1);
    for (int b = blockIdx.y; b < P.batch; b += gridDim.y) {
        const double* x = P.X + (int64_t)b * P.ldx;
        double acc = 0.0, y = 0.0;
        long long cur = -1;
        for (int e = e0; e < e1; ++e) {
            const double v = P.vals64 ? __ldg(P.vals64 + e) : (double)__ldg(P.vals + e);
            const int c = __ldg(P.col_idx + e);
            if (P.chunk > 0 && c / P.chunk != cur) {  // the reference's per-thread partials (inc/sparse.hpp:243-258)
                y = __dadd_rn(y, acc);
                acc = 0.0;
                cur = c / P.chunk;
            }
            acc = __dadd_rn(acc, __dmul_rn(v, __ldg(x + c)));
        }
        P.Y[(int64_t)b * P.ldy + r] = P.chunk > 0 ? __dadd_rn(y, acc) : acc;
    }
}

cudaError_t launch_spmm_f64(const F64Params& fp, cudaStream_t st) {
    const int gx = (fp.rows + 255) / 256;
    const int gy = fp.batch < 65535 ? fp.batch : 65535;
    csr_spmm_f64<<<dim3(gx, gy), 256, 0, st>>>(fp);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(256) csr_spmm_generic(const GenericParams P) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= P.rows) return;
    const int e0 = __ldg(P.row_ptr + r), e1 = __ldg(P.row_ptr + r + 1);
    for (int b = blockIdx.y; b < P.batch; b += gridDim.y) {
        const float* x = P.X + (int64_t)b * P.ldx;
        float acc = 0.0f;
        for (int e = e0; e < e1; ++e)
            acc = fmaf(__ldg(P.vals + e), __ldg(x + __ldg(P.col_idx + e)), acc);
        P.Y[(int64_t)b * P.ldy + r] = acc;
    }
}

// Latency-oriented SpMV / small-batch SpMM for any CSR whose rows hold at most
// KMAX entries: thread per row, every (col, val) of the row requested at once
// (fully unrolled, predicated), then every x gather at once -- three dependent
// memory round trips per row instead of one per entry.  Used for batch <= 2
// (BASELINE config 2 is a single 512^2 image: ~15 MB, latency-bound).
template <int KMAX>
__global__ void __launch_bounds__(256) csr_spmv_unrolled(const GenericParams P) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= P.rows) return;
    const int e0 = __ldg(P.row_ptr + r);
    const int cnt = __ldg(P.row_ptr + r + 1) - e0;
    if (cnt > KMAX) __trap();  // dispatcher guarantees max row length <= KMAX
    int c[KMAX];
    float v[KMAX];
#pragma unroll
    for (int q = 0; q < KMAX; ++q) {
        c[q] = q < cnt ? __ldg(P.col_idx + e0 + q) : 0;
        v[q] = q < cnt ? __ldg(P.vals + e0 + q) : 0.0f;
    }
    for (int b = 0; b < P.batch; ++b) {
        const float* x = P.X + (int64_t)b * P.ldx;
        float xv[KMAX];
#pragma unroll
        for (int q = 0; q < KMAX; ++q) xv[q] = q < cnt ? __ldg(x + c[q]) : 0.0f;
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q < KMAX; ++q)
            if (q < cnt) acc = fmaf(v[q], xv[q], acc);
        P.Y[(int64_t)b * P.ldy + r] = acc;
    }
}

cudaError_t launch_spmv_unrolled(const GenericParams& gp, int kmax, cudaStream_t st) {
    const int block = 256;
    const int grid = (gp.rows + block - 1) / block;
    if (kmax <= 9) csr_spmv_unrolled<9><<<grid, block, 0, st>>>(gp);
    else if (kmax <= 25) csr_spmv_unrolled<25><<<grid, block, 0, st>>>(gp);
    else if (kmax <= 49) csr_spmv_unrolled<49><<<grid, block, 0, st>>>(gp);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

// Latency SpMV / 2-vector SpMM (BASELINE config 2: one 512^2 image, ~15 MB):
// a warp owns 32 consecutive rows.  Their (col, val) pairs are one contiguous
// run [row_ptr[r0], row_ptr[r0+32]) that the warp streams with coalesced
// loads into shared memory; then each lane walks its own row from shared
// memory (lane stride = row length, conflict-free for odd lengths), issues
// all of the row's x gathers at once (consecutive output pixels gather
// neighbouring pixels: coalesced) and accumulates sequentially,
// acc = fmaf(val, x, acc) in stored order -- the reference's row loop, bit for
// bit.  For conv transforms with dense taps (SPEC) the run's bounds are
// predicted in closed form (row (x, y) starts at CX(x)*SY + cx(x)*CY(y)), so
// the run is requested together with row_ptr (two dependent memory trips per
// row instead of three); the loaded row_ptr decides, a mismatch reloads.
// a / s for a >= 0 with the common strides specialised (s is warp-uniform).
__device__ __forceinline__ int div_stride(int a, int s) {
    switch (s) {
        case 1: return a;
        case 2: return a >> 1;
        case 3: return a / 3;
        case 4: return a >> 2;
        default: return a / s;
    }
}

__device__ __forceinline__ int slides_before_dev(int x, int j, int dim, int s, int p) {
    const int lo = (p - j <= 0) ? 0 : div_stride(p - j + s - 1, s);
    const int hi = (dim + p - j - 1 < 0) ? 0 : div_stride(dim + p - j - 1, s) + 1;
    return max(0, min(x, hi) - lo);
}

__device__ __forceinline__ int conv_row_start(const SpecParams& P, int r) {
    if (r >= P.rows) return P.nnz;
    const int x = r / P.no, y = r - x * P.no;
    const int jlo = min(max(0, P.p - P.s * x), P.k), jhi = max(jlo, min(P.k, P.m + P.p - P.s * x));
    int cxb = 0, cyb = 0;
    for (int j = 0; j < P.k; ++j) {
        cxb += slides_before_dev(x, j, P.m, P.s, P.p);
        cyb += slides_before_dev(y, j, P.n, P.s, P.p);
    }
    return cxb * P.sy + (jhi - jlo) * cyb + P.skew;
}

// Bulk-staged latency SpMV: per warp, ONE elected lane issues three 1-D bulk
// copies (cp.async.bulk, completing on an mbarrier): row_ptr[r0 .. r0+32] and
// the (col, val) run of the warp's 32 rows.  For conv transforms with dense
// taps (SPEC) the run's bounds are closed-form, so all three copies leave at
// once, with no dependent load; otherwise row_ptr[r0], row_ptr[r0+32] are
// read first.  The copied row_ptr decides: a mismatch (test hook `skew`, or a
// matrix that is not its geometry's transform) takes a per-lane reload from
// global memory.  Programmatic dependent launch: the matrix loads are issued
// before griddepcontrol.wait, the x gathers and y stores after it, so a
// PDL-launched SpMV overlaps its matrix fetch with the previous kernel.
__device__ __forceinline__ void bulk_g2s_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Both bounds of a warp's run at once, lane-parallel: lanes 0..15 work on row
// ra, lanes 16..31 on row rb, lane j of a half on tap index j (k <= 16); two
// 16-lane reductions replace the 2 x k sequential slides_before terms.
__device__ __forceinline__ void conv_run_bounds(const SpecParams& P, int ra, int rb, int& Ea, int& Eb) {
    const int lane = threadIdx.x & 31;
    const int j = lane & 15;
    const int r = lane < 16 ? ra : rb;
    const int rr = min(r, P.rows - 1);
    const int x = rr / P.no, y = rr - x * P.no;
    const int jlo = min(max(0, P.p - P.s * x), P.k), jhi = max(jlo, min(P.k, P.m + P.p - P.s * x));
    int tx = 0, ty = 0;
    if (j < P.k) {
        tx = slides_before_dev(x, j, P.m, P.s, P.p);
        ty = slides_before_dev(y, j, P.n, P.s, P.p);
        if (P.zt) {  // zero taps: W[j] * sbx(j) + nzcol(x, i = j) * sby(i), one term per lane
            int nzc = 0;
            for (int jj = jlo; jj < jhi; ++jj) nzc += (int)((P.nzmask >> (jj * P.k + j)) & 1ull);
            tx = (int)P.zw[j] * tx + nzc * ty;
            ty = 0;
        }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
        tx += __shfl_xor_sync(0xffffffffu, tx, o);
        ty += __shfl_xor_sync(0xffffffffu, ty, o);
    }
    const int E = r >= P.rows ? P.nnz : (P.zt ? tx : tx * P.sy + (jhi - jlo) * ty) + P.skew;
    Ea = __shfl_sync(0xffffffffu, E, 0);
    Eb = __shfl_sync(0xffffffffu, E, 16);
}

template <int KMAX>
struct BulkCfg {
    static constexpr int WARPS = 4;
    static constexpr int RUN = 32 * KMAX;                 // max entries of a 32-row run
    static constexpr int BUFW = (RUN + 3 + 3) / 4 * 4;    // + 16-byte alignment slack
    static constexpr int RPW = 40;                        // 33 row_ptr words + slack
    static constexpr size_t WARP_BYTES = (size_t)(RPW + 2 * BUFW) * 4;
    static constexpr size_t SMEM = 128 + WARPS * WARP_BYTES;
};

template <int KMAX, bool SPEC, bool BULK>
__global__ void __launch_bounds__(128) csr_spmv_bulk(const SpecParams P) {
    using C = BulkCfg<KMAX>;
    extern __shared__ __align__(128) unsigned char smem[];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r0 = (blockIdx.x * C::WARPS + warp) * 32;
    if (r0 >= P.rows) return;  // warp-uniform; no block-wide barrier follows
    const int nr = min(32, P.rows - r0);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + warp;
    int* rp = reinterpret_cast<int*>(smem + 128 + (size_t)warp * C::WARP_BYTES);
    int* cb = rp + C::RPW;
    float* vb = reinterpret_cast<float*>(cb + C::BUFW);

    int E0, E1;
    bool issue;
    if (SPEC) {
        conv_run_bounds(P, r0, r0 + nr, E0, E1);
        issue = E0 >= 0 && E1 >= E0 && E1 - E0 <= C::RUN && E1 <= P.nnz;
    } else {
        E0 = __ldg(P.row_ptr + r0);
        E1 = __ldg(P.row_ptr + r0 + nr);
        if (E1 - E0 > C::RUN) __trap();  // dispatcher guarantees rows of <= KMAX entries
        issue = true;
    }
    const int rbase = r0 & ~3;
    const uint32_t rwords = (uint32_t)((r0 + nr + 1 - rbase + 3) & ~3);
    const int ebase = E0 & ~3;
    const uint32_t ewords = issue && E1 > E0 ? (uint32_t)((E1 - ebase + 3) & ~3) : 0u;
    if (BULK) {  // one elected lane, three bulk copies on an mbarrier
        if (lane == 0) {
            mbar_init(bar, 1);
            mbar_fence_init();
            mbar_expect_tx(bar, 4u * (rwords + 2u * ewords));
            bulk_g2s_1d(rp, P.row_ptr + rbase, 4u * rwords, bar);
            if (ewords) {
                bulk_g2s_1d(cb, P.col_idx + ebase, 4u * ewords, bar);
                bulk_g2s_1d(vb, P.vals + ebase, 4u * ewords, bar);
            }
        }
        __syncwarp();
        mbar_wait(bar, 0);
    } else {  // every lane: 16-byte loads, all in flight, then shared stores
        constexpr int NV = (C::BUFW / 4 + 31) / 32;
        const int nv = (int)(ewords >> 2);
        int4 cr[NV], vr[NV];
#pragma unroll
        for (int u = 0; u < NV; ++u) {
            const int q = lane + 32 * u;
            if (q < nv) {
                cr[u] = __ldg(reinterpret_cast<const int4*>(P.col_idx + ebase) + q);
                vr[u] = __ldg(reinterpret_cast<const int4*>(P.vals + ebase) + q);
            }
        }
        const int rq = (int)(rwords >> 2);
        int4 rr = lane < rq ? __ldg(reinterpret_cast<const int4*>(P.row_ptr + rbase) + lane) : make_int4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < NV; ++u) {
            const int q = lane + 32 * u;
            if (q < nv) {
                reinterpret_cast<int4*>(cb)[q] = cr[u];
                reinterpret_cast<int4*>(vb)[q] = vr[u];
            }
        }
        if (lane < rq) reinterpret_cast<int4*>(rp)[lane] = rr;
        __syncwarp();
    }
    const int* rps = rp + (r0 & 3);
    const bool hit = issue && rps[0] == E0 && rps[nr] == E1;
    if (lane >= nr) return;
    const int a = rps[lane], cnt = rps[lane + 1] - a;
    int c[KMAX];
    float v[KMAX];
    if (hit) {
        const int d0 = a - (E0 & ~3);
#pragma unroll
        for (int q = 0; q < KMAX; ++q) {
            c[q] = q < cnt ? cb[d0 + q] : 0;
            v[q] = q < cnt ? vb[d0 + q] : 0.0f;
        }
    } else {
        if (cnt > KMAX) __trap();
#pragma unroll
        for (int q = 0; q < KMAX; ++q) {
            c[q] = q < cnt ? __ldg(P.col_idx + a + q) : 0;
            v[q] = q < cnt ? __ldg(P.vals + a + q) : 0.0f;
        }
    }
    // x may be the previous kernel's output: everything below waits for it.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int bi = 0; bi < P.batch; ++bi) {
        const float* X = P.X + (int64_t)bi * P.ldx;
        float xv[KMAX];
#pragma unroll
        for (int q = 0; q < KMAX; ++q) xv[q] = q < cnt ? __ldg(X + c[q]) : 0.0f;
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q < KMAX; ++q)
            if (q < cnt) acc = fmaf(v[q], xv[q], acc);
        P.Y[(int64_t)bi * P.ldy + r0 + lane] = acc;
    }
}

// Windowed latency SpMV (conv transforms, batch <= 2): ONE memory round trip.
// csr_spmv_bulk stages a warp's matrix run, then gathers x through the staged
// columns -- two dependent trips.  Here every lane issues cp.async 16-byte
// copies of its share of the warp's row_ptr / (col, val) run (closed-form
// bounds) AND of the input window the warp's 32 outputs read: k input rows x
// (31 s + k) columns per image, addresses closed-form too -- all in flight
// together.  Each lane then walks its row from shared memory: an entry whose
// column lies in the window reads x there, any other (a matrix that is not its
// geometry's transform) reads x from global memory, so the sums are the
// per-entry ordered fmaf chain whatever the matrix holds.  Under programmatic
// dependent launch the matrix copies leave before griddepcontrol.wait, the
// window copies right after it.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int K, int S>
struct WinCfg {
    static constexpr int KK = K * K;
    static constexpr int RUN = 32 * KK;                   // max entries of a 32-row run
    static constexpr int BUFW = (RUN + 3 + 3) / 4 * 4;
    static constexpr int RPW = 40;
    static constexpr int WC = (S * 31 + K + 3 + 3) / 4 * 4;  // window columns (+ 16-byte alignment slack)
    static constexpr int WINF = 2 * K * WC;                   // two images
    static constexpr int WARPS = 4;
    static constexpr size_t WARP_BYTES = (size_t)(RPW + 2 * BUFW + WINF) * 4;
    static constexpr size_t SMEM = 128 + WARPS * WARP_BYTES;
};

template <int K, int S>
__global__ void __launch_bounds__(128) conv_spmv_win(const SpecParams P) {
    using W = WinCfg<K, S>;
    extern __shared__ __align__(128) unsigned char smem[];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r0 = (blockIdx.x * W::WARPS + warp) * 32;
    if (r0 >= P.rows) return;  // warp-uniform; no block-wide barrier follows
    const int nr = min(32, P.rows - r0);
    int* rp = reinterpret_cast<int*>(smem + 128 + (size_t)warp * W::WARP_BYTES);
    int* cb = rp + W::RPW;
    float* vb = reinterpret_cast<float*>(cb + W::BUFW);
    float* win = vb + W::BUFW;

    int E0, E1;
    conv_run_bounds(P, r0, r0 + nr, E0, E1);
    const bool issue = E0 >= 0 && E1 >= E0 && E1 - E0 <= W::RUN && E1 <= P.nnz;
    const int rbase = r0 & ~3;
    const int rq = (r0 + nr + 1 - rbase + 3) >> 2;
    const int ebase = E0 & ~3;
    const int nv = issue && E1 > E0 ? (E1 - ebase + 3) >> 2 : 0;
    // the matrix run: 16-byte loads into registers (all in flight), stored
    // to shared memory once they land (below)
    constexpr int NV = (W::BUFW / 4 + 31) / 32;
    int4 cr[NV], vr[NV];
#pragma unroll
    for (int u = 0; u < NV; ++u) {
        const int q = lane + 32 * u;
        if (q < nv) {
            cr[u] = __ldg(reinterpret_cast<const int4*>(P.col_idx + ebase) + q);
            vr[u] = __ldg(reinterpret_cast<const int4*>(P.vals + ebase) + q);
        }
    }
    const int4 rr = lane < rq ? __ldg(reinterpret_cast<const int4*>(P.row_ptr + rbase) + lane) : make_int4(0, 0, 0, 0);
    // the input window of the warp's first output-row segment: K input rows
    const int x = r0 / P.no, y0 = r0 - x * P.no;
    const int wa0 = S * x - P.p;                          // input row of tap row 0
    const int c0 = max(S * y0 - P.p, 0) & ~3;             // first window column (16-byte aligned)
    const int c1 = min(S * (y0 + 31) + K - 1 - P.p, P.n - 1);
    const int nq = c1 >= c0 ? min((c1 - c0) / 4 + 1, W::WC / 4) : 0;  // 16-byte units per row
    // x may be the previous kernel's output: the window copies wait for it.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int bi = 0; bi < P.batch; ++bi) {
        const float* Xb = P.X + (int64_t)bi * P.ldx + c0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int a = wa0 + j;
            if (a >= 0 && a < P.m)
                for (int q = lane; q < nq; q += 32)
                    cp_async16(win + (bi * K + j) * W::WC + 4 * q, Xb + (int64_t)a * P.n + 4 * q);
        }
    }
#pragma unroll
    for (int u = 0; u < NV; ++u) {
        const int q = lane + 32 * u;
        if (q < nv) {
            reinterpret_cast<int4*>(cb)[q] = cr[u];
            reinterpret_cast<int4*>(vb)[q] = vr[u];
        }
    }
    if (lane < rq) reinterpret_cast<int4*>(rp)[lane] = rr;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    const int* rps = rp + (r0 & 3);
    const bool hit = issue && rps[0] == E0 && rps[nr] == E1;
    if (lane >= nr) return;
    const int y = y0 + lane;
    int a0, cnt;
    const int* cs;
    const float* vs;
    if (hit) {
        a0 = rps[lane];
        cnt = rps[lane + 1] - a0;
        cs = cb + (a0 - ebase);
        vs = vb + (a0 - ebase);
    } else {
        a0 = __ldg(P.row_ptr + r0 + lane);
        cnt = __ldg(P.row_ptr + r0 + lane + 1) - a0;
        cs = P.col_idx + a0;
        vs = P.vals + a0;
    }
    // A row of this warp's output-row segment whose K x K taps all land reads
    // its entries' x from the window when their columns are the pattern's.
    const bool full = hit && y < P.no && cnt == W::KK && S * x - P.p >= 0 && S * x - P.p + K <= P.m &&
                      S * y - P.p >= 0 && S * y - P.p + K <= P.n;
    const int colb = (S * x - P.p) * P.n + (S * y - P.p);   // column of tap (0, 0)
    const int wcol = S * y - P.p - c0;                       // its window column
    for (int bi = 0; bi < P.batch; ++bi) {
        const float* X = P.X + (int64_t)bi * P.ldx;
        const float* wb = win + bi * K * W::WC;
        float acc = 0.0f;
        if (full) {
            float xv[W::KK], vv[W::KK];
            bool pat = true;
#pragma unroll
            for (int q = 0; q < W::KK; ++q) {
                const int j = q / K, i = q % K;
                const int c = cs[q];
                pat &= c == colb + j * P.n + i;
                vv[q] = vs[q];
                xv[q] = wb[j * W::WC + wcol + i];
            }
            if (pat) {
#pragma unroll
                for (int q = 0; q < W::KK; ++q) acc = fmaf(vv[q], xv[q], acc);
            } else {
                for (int q = 0; q < W::KK; ++q) acc = fmaf(vv[q], __ldg(X + cs[q]), acc);
            }
        } else {
            for (int q = 0; q < cnt; ++q) acc = fmaf(vs[q], __ldg(X + cs[q]), acc);
        }
        P.Y[(int64_t)bi * P.ldy + r0 + lane] = acc;
    }
}

template <int K, int S>
static cudaError_t launch_win_ks(const SpecParams& sp, cudaStream_t st) {
    using W = WinCfg<K, S>;
    static std::atomic<bool> attr_set[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(conv_spmv_win<K, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)W::SMEM);
        if (e != cudaSuccess) return e;
        attr_set[dev & 63] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((sp.rows + 32 * W::WARPS - 1) / (32 * W::WARPS)));
    cfg.blockDim = dim3(32 * W::WARPS);
    cfg.dynamicSmemBytes = W::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = sp.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, conv_spmv_win<K, S>, sp);
}

// The windowed kernel: conv transforms (closed-form runs) of the instantiated
// (k, s) -- the BASELINE and DenseNet121 geometries -- whose window rows are
// 16-byte aligned (n, ldx multiples of 4, X aligned).
bool spmv_win_ok(const SpecParams& sp) {
    const bool ks = (sp.s == 1 && (sp.k == 1 || sp.k == 3 || sp.k == 5 || sp.k == 7)) ||
                    (sp.s == 2 && (sp.k == 2 || sp.k == 3 || sp.k == 5 || sp.k == 7));
    return ks && sp.n % 4 == 0 && sp.ldx % 4 == 0 && reinterpret_cast<uintptr_t>(sp.X) % 16 == 0;
}

cudaError_t launch_spmv_win(const SpecParams& sp, int kmax, cudaStream_t st) {
    (void)kmax;
    if (sp.batch < 1 || sp.batch > 2 || !spmv_win_ok(sp)) return cudaErrorInvalidValue;
    if (sp.s == 1) {
        switch (sp.k) {
            case 1: return launch_win_ks<1, 1>(sp, st);
            case 3: return launch_win_ks<3, 1>(sp, st);
            case 5: return launch_win_ks<5, 1>(sp, st);
            case 7: return launch_win_ks<7, 1>(sp, st);
        }
    } else {
        switch (sp.k) {
            case 2: return launch_win_ks<2, 2>(sp, st);
            case 3: return launch_win_ks<3, 2>(sp, st);
            case 5: return launch_win_ks<5, 2>(sp, st);
            case 7: return launch_win_ks<7, 2>(sp, st);
        }
    }
    return cudaErrorInvalidValue;
}

template <int KMAX>
static cudaError_t launch_bulk_k(const SpecParams& sp, bool spec, cudaStream_t st) {
    using C = BulkCfg<KMAX>;
    // staging: per-lane 16-byte loads (default; config 2 14.6 vs 16.0 us, DenseNet
    // table 144 vs 151 us, profiles/r01l) or bulk copies (option stage=bulk)
    const bool bulk = opt(kOptStage) == 1;
    auto kern = spec ? (bulk ? csr_spmv_bulk<KMAX, true, true> : csr_spmv_bulk<KMAX, true, false>)
                     : (bulk ? csr_spmv_bulk<KMAX, false, true> : csr_spmv_bulk<KMAX, false, false>);
    static std::atomic<bool> attr_set[4][64];
    int dev = 0;
    cudaGetDevice(&dev);
    const int which = (spec ? 2 : 0) + (bulk ? 1 : 0);
    if (!attr_set[which][dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e != cudaSuccess) return e;
        attr_set[which][dev & 63] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((sp.rows + 32 * C::WARPS - 1) / (32 * C::WARPS)));
    cfg.blockDim = dim3(32 * C::WARPS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = sp.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, sp);
}

cudaError_t launch_spmv_warp(const SpecParams& sp, int kmax, bool spec, cudaStream_t st) {
    if (sp.batch < 1 || sp.batch > 2) return cudaErrorInvalidValue;
    if (kmax <= 9) return launch_bulk_k<9>(sp, spec, st);
    if (kmax <= 25) return launch_bulk_k<25>(sp, spec, st);
    if (kmax <= 49) return launch_bulk_k<49>(sp, spec, st);
    return cudaErrorInvalidValue;
}

template <int BT>
static cudaError_t launch_bt(const TiledParams& tp, const CUtensorMap* tmap, size_t smem,
                             cudaStream_t st) {
    static std::atomic<bool> attr_set[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(conv_spmm_tiled<BT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set[dev & 63] = true;
    }
    const int tiles_x = (tp.mo + tp.th - 1) / tp.th;
    const int grid = tiles_x * tp.tiles_y;
    conv_spmm_tiled<BT><<<grid, tp.th * kTileW, smem, st>>>(*tmap, tp);
    return cudaGetLastError();
}

cudaError_t launch_tiled(const TiledParams& tp, const CUtensorMap* tmap, int bt, size_t smem,
                         cudaStream_t st) {
    switch (bt) {
        case 1: return launch_bt<1>(tp, tmap, smem, st);
        case 2: return launch_bt<2>(tp, tmap, smem, st);
        case 4: return launch_bt<4>(tp, tmap, smem, st);
        case 8: return launch_bt<8>(tp, tmap, smem, st);
        default: return cudaErrorInvalidValue;
    }
}

// Multi-vector SpMM for any CSR whose rows hold at most `kmax` entries (the
// generic path of matrices that are not conv transforms -- read_sparse,
// uploads -- and of forced runs): a CTA owns 128 consecutive rows, stages
// their (col, val) run in shared memory ONCE with coalesced loads, then walks
// its share of the batch, IMG images at a time, each thread accumulating its
// row in stored order (acc = fmaf(val, x[col], acc), bit-exact with the
// per-row loop).  The matrix is read once per CTA (per image group) instead
// of once per image.
template <int IMG>
__global__ void __launch_bounds__(128) csr_spmm_rowblock(const GenericParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int t = threadIdx.x;
    const int r0 = blockIdx.x * 128;
    const int r1 = min(P.rows, r0 + 128);
    const int e0 = __ldg(P.row_ptr + r0), e1 = __ldg(P.row_ptr + r1);
    int* sc = reinterpret_cast<int*>(smem);
    float* sv = reinterpret_cast<float*>(sc + P.stage_cap);
    for (int e = e0 + t; e < e1; e += 128) {
        sc[e - e0] = __ldg(P.col_idx + e);
        sv[e - e0] = __ldg(P.vals + e);
    }
    __syncthreads();
    const int r = r0 + t;
    if (r >= r1) return;
    const int a = __ldg(P.row_ptr + r) - e0, b = __ldg(P.row_ptr + r + 1) - e0;
    // images in groups of IMG: group blockIdx.y, blockIdx.y + gridDim.y, ...
    for (int i0 = blockIdx.y * IMG; i0 < P.batch; i0 += gridDim.y * IMG) {
        const int ni = min(IMG, P.batch - i0);
        // per-image row pointers once per group (images past the batch alias
        // the first: their sums are computed and dropped), so a gather is one
        // address multiply-add and the load -- no 64-bit index arithmetic and
        // no predicates in the entry loop
        const float* xq[IMG];
#pragma unroll
        for (int q = 0; q < IMG; ++q) xq[q] = P.X + (int64_t)(i0 + (q < ni ? q : 0)) * P.ldx;
        float acc[IMG];
#pragma unroll
        for (int q = 0; q < IMG; ++q) acc[q] = 0.0f;
        for (int e = a; e < b; ++e) {
            const int c = sc[e];
            const float v = sv[e];
#pragma unroll
            for (int q = 0; q < IMG; ++q) acc[q] = fmaf(v, __ldg(xq[q] + c), acc[q]);
        }
#pragma unroll
        for (int q = 0; q < IMG; ++q)
            if (q < ni) P.Y[(int64_t)(i0 + q) * P.ldy + r] = acc[q];
    }
}

template <int IMG>
static cudaError_t launch_rowblock_i(const GenericParams& gp, size_t smem, cudaStream_t st) {
    static std::atomic<bool> attr[64];
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (smem > 48 * 1024 && !attr[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(csr_spmm_rowblock<IMG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             64 * 1024);
        if (e != cudaSuccess) return e;
        attr[dev & 63] = true;
    }
    const int gx = (gp.rows + 127) / 128;
    // enough CTAs for every SM several times over; each reads the matrix once
    const int groups = (gp.batch + IMG - 1) / IMG;
    const int gy = std::max(1, std::min(groups, (sms * 16 + gx - 1) / gx));
    csr_spmm_rowblock<IMG><<<dim3(gx, std::min(gy, 65535)), 128, smem, st>>>(gp);
    return cudaGetLastError();
}

cudaError_t launch_rowblock(GenericParams gp, int kmax, cudaStream_t st) {
    if (kmax > 64) return cudaErrorInvalidValue;
    gp.stage_cap = 128 * std::max(kmax, 1);
    const size_t smem = (size_t)gp.stage_cap * 8;
    // images per group: 8 (config 3 shape as a generic CSR, 256 images:
    // 1.41 / 1.48 / 1.15 / 1.69 ms for 2 / 4 / 8 / 16, profiles/r01_generic)
    return launch_rowblock_i<8>(gp, smem, st);
}

cudaError_t launch_generic(const GenericParams& gp, cudaStream_t st) {
    const int block = 256;
    const int gx = (gp.rows + block - 1) / block;
    const int gy = gp.batch < 65535 ? gp.batch : 65535;
    csr_spmm_generic<<<dim3(gx, gy), block, 0, st>>>(gp);
    return cudaGetLastError();
}

}  // namespace spb
