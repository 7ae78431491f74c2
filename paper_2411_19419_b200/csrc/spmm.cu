// spmm.cu -- SpMV / SpMM of the conv transform T against image-major batches.
//
// Replaces spmv + detail::spmv_csr_rows (inc/sparse.hpp:180-192, 214-261) and
// the per-image convolve loop of its callers (inc/conv.hpp:207-215,
// inc/bench.hpp:240-248).  Accumulation contract, both kernels:
//     acc = +0.0f; for e in row (column-ascending): acc = fmaf(val[e], x[col[e]], acc)
// i.e. the reference's sequential row loop in fp32 with one rounding per step.
//
// conv_spmm_tiled -- the hot path for transforms built by csr_build.  A CTA owns
//   a TH x 32 block of output pixels (TH*32 rows of T; warp w = one image row
//   of the block, lane = one output column).  Prologue: each thread reads its
//   row's (col, val) pairs from the CSR ONCE and rewrites every column as an
//   offset into the CTA's input window (the (TH-1)s+k x 31s+k patch every
//   entry of the block falls in); the pairs live tap-major in shared memory
//   ([q][thread], bank-conflict free).  Main loop: the input window of BT
//   images at a time is staged into shared memory by one TMA 3-D box load
//   (cols x rows x images; negative / out-of-range coordinates zero-fill,
//   so padding costs nothing), multi-buffered on mbarriers, and every thread
//   accumulates its row for BT images from shared memory.  HBM traffic: the
//   matrix once per launch, each input image once (+ window halo from L2),
//   each output once; per CTA the CSR is read once per batch, not per image.
// csr_spmm_generic -- any CSR (uploaded host matrices, misfit geometries):
//   thread per (row, image), x gathered through L1.
#include "internal.h"

namespace spb {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

constexpr int kTileW = 32;

}  // namespace

size_t tiled_smem_bytes(int th, int wr, int wc, int k2max, int bt, int stages) {
    const size_t bars = 128;  // mbarriers, padded so the windows stay 128B-aligned
    const size_t win = (size_t)stages * bt * wr * wc * sizeof(float);
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

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    float* xs = reinterpret_cast<float*>(smem + 128);
    int32_t* s_off = reinterpret_cast<int32_t*>(xs + (size_t)stages * BT * win);
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
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap))
                     : "memory");
        for (int st = 0; st < stages; ++st) mbar_init(&bars[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t bytes = (uint32_t)(BT * win * sizeof(float));
        for (int st = 0; st < stages && st < G; ++st) {
            mbar_expect_tx(&bars[st], bytes);
            tma_load_3d(xs + (size_t)st * BT * win, &tmap, wc0, wr0, st * BT, &bars[st]);
        }
    }

    // Prologue: this row's CSR entries -> window offsets, tap-major in smem.
    int cnt = 0;
    if (valid) {
        const int e0 = __ldg(P.row_ptr + r);
        cnt = __ldg(P.row_ptr + r + 1) - e0;
        if (cnt > P.k2max) __trap();
        for (int q = 0; q < cnt; ++q) {
            const int c = __ldg(P.col_idx + e0 + q);
            const float v = __ldg(P.vals + e0 + q);
            const int ri = c / P.n;
            const int dr = ri - wr0, dc = c - ri * P.n - wc0;
            if ((unsigned)dr >= (unsigned)P.wr || (unsigned)dc >= (unsigned)P.wc) __trap();
            s_off[q * TILE + t] = dr * P.wc + dc;
            s_val[q * TILE + t] = v;
        }
    }
    __syncthreads();  // mbarrier init visible to all waiters

    for (int g = 0; g < G; ++g) {
        const int st = g % stages;
        float* xw = xs + (size_t)st * BT * win;
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
            const int off = s_off[q * TILE + t];
            const float v = s_val[q * TILE + t];
#pragma unroll
            for (int b = 0; b < BT; ++b) acc[b] = fmaf(v, xw[b * win + off], acc[b]);
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

__global__ void __launch_bounds__(256) csr_spmm_generic(const GenericParams P) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= P.rows) return;
    const int e0 = __ldg(P.row_ptr + r), e1 = __ldg(P.row_ptr + r + 1);
    for (int b = blockIdx.y; b < P.batch; b += gridDim.y) {
        const float* x = P.X + (int64_t)b * P.ldx;
        float acc = 0.0f;
        for (int e = e0; e < e1; ++e) acc = fmaf(__ldg(P.vals + e), __ldg(x + __ldg(P.col_idx + e)), acc);
        P.Y[(int64_t)b * P.ldy + r] = acc;
    }
}

template <int BT>
static cudaError_t launch_bt(const TiledParams& tp, const CUtensorMap* tmap, size_t smem,
                             cudaStream_t st) {
    static bool attr_set[64] = {};
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

cudaError_t launch_generic(const GenericParams& gp, cudaStream_t st) {
    const int block = 256;
    const int gx = (gp.rows + block - 1) / block;
    const int gy = gp.batch < 65535 ? gp.batch : 65535;
    csr_spmm_generic<<<dim3(gx, gy), block, 0, st>>>(gp);
    return cudaGetLastError();
}

}  // namespace spb
