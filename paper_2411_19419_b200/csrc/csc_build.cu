// csc_build.cu -- one-pass on-device construction of T = C*P in CSC layout.
//
// Replaces build_transform(kernel, spec, Layout::CSC) (inc/conv.hpp:179-204,
// compile with layout CSC at inc/sparse.hpp:85-119) and relayout(T, CSC)
// (inc/sparse.hpp:268-274) for conv transforms.  Like the CSR build, nothing
// is sorted: each column's entries are generated in their final order.
//
// Column c = a*n + b is input pixel (a, b).  Output row (x, y) stores it with
// tap (j, i) iff s*x + j - p = a and s*y + i - p = b, i.e.
//   j in J(a) = { j in [0, k) : j == (a + p) mod s,  x = (a + p - j)/s in [0, m_out) }
// (and I(b) alike), and the tap is not an exact zero (inc/sparse.hpp:335).
// Rows ascend with x then y, i.e. with j DEScending then i descending.
//
// col_ptr is closed-form.  With NI[i] = #{y : 0 <= s*y + i - p < n} and
// RT[j] = sum_i nz[j][i] * NI[i], the entries in all columns before (a, b) are
//   sum_j RT[j] * #{x : 0 <= s*x + j - p < a}
//     + sum_{j in J(a)} sum_i nz[j][i] * #{y : 0 <= s*y + i - p < b},
// every count an O(1) range, so a CTA finds its global offset in O(k^2) without
// a grid-wide scan; a block scan of the per-column counts finishes col_ptr.
// Entries are staged in shared memory at the global offset's 16-byte phase and
// streamed out with vector stores (as csr_build.cu does).
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

// #{x in [0, mo) : lo <= s*x + j - p < hi}
__device__ __forceinline__ int slide_count(int j, int lo, int hi, int mo, int s, int p) {
    if (hi <= lo) return 0;
    const int a = lo + p - j;      // s*x >= a
    const int b = hi - 1 + p - j;  // s*x <= b
    if (b < 0) return 0;
    const int xlo = a <= 0 ? 0 : (a + s - 1) / s;
    const int xhi = min(mo - 1, b / s);
    return max(0, xhi - xlo + 1);
}

// Taps landing on input coordinate a: j = jtop, jtop - s, ... > jbot (x ascending).
__device__ __forceinline__ void tap_set(int a, int k, int s, int p, int mo, int& jtop, int& jbot) {
    const int ap = a + p;
    int top = min(k - 1, ap);
    top -= ((top - ap) % s + s) % s;  // top == ap (mod s)
    jtop = top;
    jbot = ap - s * mo;  // j > jbot  <=>  x < mo
}

}  // namespace

// KC = compile-time kernel side (0: runtime P.k); DENSE: no zero taps.
template <int KC, bool DENSE>
__global__ void __launch_bounds__(256) csc_build_kernel(const CscParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_warp[32];
    __shared__ long long s_base;
    const int t = threadIdx.x, R = blockDim.x, nw = R >> 5, lane = t & 31, wid = t >> 5;
    const int k = KC ? KC : P.k, kk = k * k, S = P.s;
    float* s_taps = reinterpret_cast<float*>(smem);
    const int tab_words = (kk + 3) & ~3;
    for (int q = t; q < kk; q += R) s_taps[q] = __ldg(P.taps + q);
    if (t == 0) s_base = 0;
    __syncthreads();

    const int c0 = blockIdx.x * R;
    const int c = c0 + t;
    // J(a) = {jtop, jtop - s, ...} down to > jlo; x runs up from x_top as j steps down
    int a = 0, b = 0, cnt = 0, jtop = -1, jlo = 0, itop = -1, ilo = 0;
    if (c < P.cols) {
        a = c / P.n;
        b = c - a * P.n;
        int jbot, ibot;
        tap_set(a, k, S, P.p, P.mo, jtop, jbot);
        tap_set(b, k, S, P.p, P.no, itop, ibot);
        jlo = max(jbot, -1);
        ilo = max(ibot, -1);
        const int nj = jtop > jlo ? (jtop - jlo - 1) / S + 1 : 0;
        const int ni = itop > ilo ? (itop - ilo - 1) / S + 1 : 0;
        if (DENSE) {
            cnt = nj * ni;
        } else {
            for (int j = jtop; j > jlo; j -= S)
                for (int i = itop; i > ilo; i -= S) cnt += s_taps[j * k + i] != 0.0f ? 1 : 0;
        }
    }

    // ---- closed-form global offset of column c0 = (a0, b0): warp 0, lanes over j ----
    if (wid == 0) {
        const int a0 = c0 / P.n, b0 = c0 - a0 * P.n;
        int jt0, jb0;
        tap_set(a0, k, S, P.p, P.mo, jt0, jb0);
        long long part = 0;
        for (int j = lane; j < k; j += 32) {
            long long rt = 0, rb = 0;
            for (int i = 0; i < k; ++i) {
                if (!DENSE && s_taps[j * k + i] == 0.0f) continue;
                rt += slide_count(i, 0, P.n, P.no, S, P.p);
                rb += slide_count(i, 0, b0, P.no, S, P.p);
            }
            part += rt * slide_count(j, 0, a0, P.mo, S, P.p);
            const bool in_a0 = j <= jt0 && j > jb0 && ((jt0 - j) % S) == 0;
            if (in_a0) part += rb;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) s_base = part;
    }

    // ---- block exclusive scan of the counts ----
    const int inc = warp_incl_scan(cnt);
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int wv = lane < nw ? s_warp[lane] : 0;
        wv = warp_incl_scan(wv);
        s_warp[lane] = wv;
    }
    __syncthreads();
    const int excl = inc - cnt + (wid > 0 ? s_warp[wid - 1] : 0);
    const int total = s_warp[nw - 1];
    const int base = (int)s_base;
    if (c < P.cols) {
        P.col_ptr[c] = base + excl;
        if (c == P.cols - 1) P.col_ptr[P.cols] = base + excl + cnt;
    }

    // ---- fill: rows ascending = j descending (x ascending), then i descending ----
    const int mis = base & 3;
    int32_t* drow;
    float* dval;
    int o;
    // compile-time for the unrolled k (always staged): shared, not generic, accesses
    const bool staged = KC > 0 || P.stage != 0;
    if (staged) {
        drow = reinterpret_cast<int32_t*>(smem) + tab_words;
        dval = reinterpret_cast<float*>(drow) + P.stage_words;
        o = mis + excl;
    } else {
        drow = P.row_idx;
        dval = P.vals;
        o = base + excl;
    }
    if (KC && DENSE && S == 1 && cnt == KC * KC) {
        // Interior column at stride 1 (every tap lands): the unrolled K x K
        // pattern, x and y stepping with j and i descending.
        const int x0 = a + P.p - (KC - 1), y0 = b + P.p - (KC - 1);
#pragma unroll
        for (int jj = 0; jj < KC; ++jj)
#pragma unroll
            for (int ii = 0; ii < KC; ++ii) {
                drow[o + jj * KC + ii] = (x0 + jj) * P.no + y0 + ii;
                dval[o + jj * KC + ii] = s_taps[(KC - 1 - jj) * KC + (KC - 1 - ii)];
            }
    } else if (c < P.cols && cnt > 0) {
        const int x0 = (a + P.p - jtop) / S, y0 = (b + P.p - itop) / S;  // exact: jtop == a+p (mod s)
        int xrow = x0 * P.no;
        for (int j = jtop; j > jlo; j -= S, xrow += P.no) {
            int y = y0;
            for (int i = itop; i > ilo; i -= S, ++y) {
                const float v = s_taps[j * k + i];
                if (DENSE || v != 0.0f) {  // drops +-0.0, keeps NaN
                    drow[o] = xrow + y;
                    dval[o] = v;
                    ++o;
                }
            }
        }
    }
    if (staged) {
        if (P.bulk_store) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        const int head = min(total, (4 - mis) & 3);
        if (t < head) {
            __stcs(P.row_idx + base + t, drow[mis + t]);
            __stcs(P.vals + base + t, dval[mis + t]);
        }
        const int nvec = (total - head) >> 2;
        const int4* srow = reinterpret_cast<const int4*>(drow + mis + head);
        const float4* sval = reinterpret_cast<const float4*>(dval + mis + head);
        int4* grow = reinterpret_cast<int4*>(P.row_idx + base + head);
        float4* gval = reinterpret_cast<float4*>(P.vals + base + head);
        if (P.bulk_store) {  // the 16-byte body through the TMA engine: two instructions
            if (t == 0 && nvec > 0) {
                bulk_s2g(grow, srow, (uint32_t)nvec * 16u);
                bulk_s2g(gval, sval, (uint32_t)nvec * 16u);
                bulk_commit_wait_read();
            }
        } else {
            for (int q = t; q < nvec; q += R) {
                __stcs(grow + q, srow[q]);
                __stcs(gval + q, sval[q]);
            }
        }
        const int done = head + 4 * nvec;
        if (t < total - done) {
            __stcs(P.row_idx + base + done + t, drow[mis + done + t]);
            __stcs(P.vals + base + done + t, dval[mis + done + t]);
        }
    }
}

// Block size and staging for a per-column maximum of `maxc` entries.
cudaError_t launch_csc_build(CscParams cp, int maxc, bool dense, cudaStream_t st) {
    const int kk = cp.k * cp.k;
    const size_t tab_bytes = (size_t)((kk + 3) & ~3) * 4;
    int block = 256;
    while (block > 64 && (size_t)block * maxc * 8 > 64 * 1024) block >>= 1;
    size_t smem = tab_bytes;
    cp.stage = 0;
    if ((size_t)block * maxc * 8 <= 96 * 1024 && tab_bytes <= 64 * 1024) {
        cp.stage = 1;
        cp.stage_words = (int)((block * maxc + 3 + 3) & ~3);
        smem += (size_t)cp.stage_words * 4 * 2;
    } else {
        block = 256;
    }
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    auto kern = csc_build_kernel<0, false>;  // (the unrolled variants assume staging)
    if (!cp.stage) {
        if (dense) kern = csc_build_kernel<0, true>;
    } else if (dense) {
        switch (cp.k) {
            case 1: kern = csc_build_kernel<1, true>; break;
            case 3: kern = csc_build_kernel<3, true>; break;
            case 5: kern = csc_build_kernel<5, true>; break;
            case 7: kern = csc_build_kernel<7, true>; break;
            case 11: kern = csc_build_kernel<11, true>; break;
            default: kern = csc_build_kernel<0, true>; break;
        }
    } else {
        switch (cp.k) {
            case 3: kern = csc_build_kernel<3, false>; break;
            case 5: kern = csc_build_kernel<5, false>; break;
            case 7: kern = csc_build_kernel<7, false>; break;
            default: break;
        }
    }
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const long long grid = (cp.cols + block - 1) / block;
    kern<<<(unsigned)grid, block, smem, st>>>(cp);
    return cudaGetLastError();
}

}  // namespace spb
