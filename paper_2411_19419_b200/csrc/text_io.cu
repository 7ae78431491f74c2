// text_io.cu -- transform persistence on the device path.
//
// write_transform (inc/conv.hpp:217-224) + write_sparse (inc/sparse.hpp:400-406):
//     %%transform m n k s p csr
//     %%sparse coordinate real
//     rows cols nnz
//     row col value            (1-based, storage order, value as "%.17g")
// The reference formats every entry on the host with snprintf; here the GPU
// renders the text: a sizing pass (bytes per block of rows), a scan of the
// block totals, and a rendering pass that stages each block's lines in shared
// memory and writes them out contiguously.  Values are fp32 widened to double
// (the reference's value type), printed with an exact %.17g: 17 significant
// digits of the binary value, correctly rounded (glibc semantics: round half
// to even on the exact value), %g's choice of fixed or exponent style,
// trailing zeros stripped, and "inf" / "-inf" / "nan" / "-nan" spellings.
// The result is byte-identical to the reference's file for the same matrix.
#include <cstring>
#include <mutex>

#include "internal.h"

namespace spb {

namespace {

__constant__ unsigned long long c_pow5[62][3];  // 5^k, k = 0..61, little-endian 64-bit limbs

// q = round_half_even(n >> rs) for a 192-bit n, rs >= 1; q < 2^64 assumed.
__device__ __forceinline__ unsigned long long shr192_round(const unsigned long long n[3], int rs) {
    auto limb = [&](int i) -> unsigned long long { return i < 3 ? n[i] : 0ull; };
    const int li = rs >> 6, bo = rs & 63;
    unsigned long long q = bo ? (limb(li) >> bo) | (limb(li + 1) << (64 - bo)) : limb(li);
    const int hb = rs - 1;
    const bool half = (limb(hb >> 6) >> (hb & 63)) & 1ull;
    bool sticky = false;
    const int sl = hb >> 6, sb = hb & 63;
    for (int i = 0; i < sl; ++i) sticky |= limb(i) != 0ull;
    if (sb) sticky |= (limb(sl) & ((1ull << sb) - 1ull)) != 0ull;
    if (half && (sticky || (q & 1ull))) ++q;
    return q;
}

// round_half_even(M * 2^E * 10^k) exactly (M < 2^24).
__device__ unsigned long long scaled_round(unsigned M, int E, int k) {
    if (k >= 0) {
        const unsigned long long* p5 = c_pow5[k];
        unsigned long long n[3];
        unsigned __int128 t = (unsigned __int128)p5[0] * M;
        n[0] = (unsigned long long)t;
        t = (t >> 64) + (unsigned __int128)p5[1] * M;
        n[1] = (unsigned long long)t;
        t = (t >> 64) + (unsigned __int128)p5[2] * M;
        n[2] = (unsigned long long)t;
        const int sh = E + k;
        if (sh >= 0) return n[0] << sh;  // exact (the caller keeps the result < 10^18)
        return shr192_round(n, -sh);
    }
    const int q = -k;  // value >= 1e17: E - q >= 0
    unsigned long long d5 = 1;
    for (int i = 0; i < q; ++i) d5 *= 5ull;
    const unsigned __int128 num = (unsigned __int128)M << (E - q);
    unsigned long long quo = (unsigned long long)(num / d5);
    const unsigned long long rem = (unsigned long long)(num - (unsigned __int128)quo * d5);
    if (2 * (unsigned __int128)rem > d5) ++quo;  // 5^q is odd: no ties
    return quo;
}

}  // namespace

// "%.17g" of (double)v into out (<= 24 chars, no terminator); returns the length.
__device__ int format_g17(float v, char* out) {
    const unsigned bits = __float_as_uint(v);
    int o = 0;
    if (bits >> 31) out[o++] = '-';
    const unsigned ex = (bits >> 23) & 0xffu, man = bits & 0x7fffffu;
    if (ex == 0xffu) {
        const char* w = man ? "nan" : "inf";
        for (int i = 0; i < 3; ++i) out[o++] = w[i];
        return o;
    }
    if (ex == 0 && man == 0) {
        out[o++] = '0';
        return o;
    }
    const unsigned M = ex ? (man | 0x800000u) : man;
    const int E = ex ? (int)ex - 150 : -149;
    int X = (int)floor(log10((double)M) + E * 0.30102999566398120);
    unsigned long long D = 0;
    for (int guard = 0; guard < 4; ++guard) {
        D = scaled_round(M, E, 16 - X);
        if (D >= 100000000000000000ull) ++X;
        else if (D < 10000000000000000ull) --X;
        else break;
    }
    char dg[17];
    for (int i = 16; i >= 0; --i) {
        dg[i] = (char)('0' + (int)(D % 10ull));
        D /= 10ull;
    }
    int last = 16;
    while (last > 0 && dg[last] == '0') --last;
    if (X >= -4 && X < 17) {
        if (X >= 0) {
            for (int i = 0; i <= X; ++i) out[o++] = dg[i];
            if (last > X) {
                out[o++] = '.';
                for (int i = X + 1; i <= last; ++i) out[o++] = dg[i];
            }
        } else {
            out[o++] = '0';
            out[o++] = '.';
            for (int i = 0; i < -X - 1; ++i) out[o++] = '0';
            for (int i = 0; i <= last; ++i) out[o++] = dg[i];
        }
    } else {
        out[o++] = dg[0];
        if (last > 0) {
            out[o++] = '.';
            for (int i = 1; i <= last; ++i) out[o++] = dg[i];
        }
        out[o++] = 'e';
        out[o++] = X < 0 ? '-' : '+';
        const int ax = X < 0 ? -X : X;
        if (ax >= 100) out[o++] = (char)('0' + ax / 100);
        out[o++] = (char)('0' + (ax / 10) % 10);
        out[o++] = (char)('0' + ax % 10);
    }
    return o;
}

// ---- "%.17g" of an arbitrary double ----------------------------------------
// Handles that keep exact fp64 values (vals64: taps or entries that fp32 does
// not represent) print them with the reference's own format.  v = M * 2^E
// exactly; D = round_half_even(v * 10^(16-X)) is computed as an exact
// quotient Num / Den of big integers (<= 1024 bits: 5^340 * 2^53 at the
// subnormal end, 2^971 * 2^53 / 5^292 at the top), so every double -- normal,
// subnormal, huge -- prints as glibc prints it.  Host + device: the CPU tests
// compare it with snprintf.
namespace {

constexpr int kBigLimbs = 17;
struct Big {
    unsigned long long w[kBigLimbs];
};

__host__ __device__ inline void big_set(Big& a, unsigned long long v) {
    a.w[0] = v;
    for (int i = 1; i < kBigLimbs; ++i) a.w[i] = 0;
}
__host__ __device__ inline void big_mul_small(Big& a, unsigned long long m) {
    unsigned __int128 c = 0;
    for (int i = 0; i < kBigLimbs; ++i) {
        c += (unsigned __int128)a.w[i] * m;
        a.w[i] = (unsigned long long)c;
        c >>= 64;
    }
}
__host__ __device__ inline void big_mul_pow5(Big& a, int q) {
    for (; q >= 27; q -= 27) big_mul_small(a, 7450580596923828125ull);  // 5^27
    unsigned long long r = 1;
    for (; q > 0; --q) r *= 5ull;
    big_mul_small(a, r);
}
__host__ __device__ inline void big_shl(Big& a, int s) {
    const int li = s >> 6, bo = s & 63;
    for (int i = kBigLimbs - 1; i >= 0; --i) {
        const unsigned long long lo = i - li >= 0 ? a.w[i - li] : 0ull;
        const unsigned long long lo2 = i - li - 1 >= 0 ? a.w[i - li - 1] : 0ull;
        a.w[i] = bo ? (lo << bo) | (lo2 >> (64 - bo)) : lo;
    }
}
__host__ __device__ inline void big_shr1(Big& a) {
    for (int i = 0; i < kBigLimbs; ++i) a.w[i] = (a.w[i] >> 1) | (i + 1 < kBigLimbs ? a.w[i + 1] << 63 : 0ull);
}
__host__ __device__ inline int big_cmp(const Big& a, const Big& b) {
    for (int i = kBigLimbs - 1; i >= 0; --i)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
}
__host__ __device__ inline void big_sub(Big& a, const Big& b) {  // a -= b (a >= b)
    unsigned long long borrow = 0;
    for (int i = 0; i < kBigLimbs; ++i) {
        const unsigned long long x = a.w[i], y = b.w[i];
        const unsigned long long d = x - y - borrow;
        borrow = (x < y) || (x - y < borrow) ? 1ull : 0ull;
        a.w[i] = d;
    }
}

// floor(M * 2^E * 10^k) (known to be < 2^64); *up = round-half-even adds one.
__host__ __device__ inline unsigned long long scaled_floor64(unsigned long long M, int E, int k, bool* up) {
    Big num, den;
    big_set(num, M);
    big_set(den, 1);
    if (k >= 0) big_mul_pow5(num, k);
    else big_mul_pow5(den, -k);
    const int t = E + k;  // power of two
    if (t >= 0) big_shl(num, t);
    else big_shl(den, -t);
    // quotient bits 63..0 by restoring division against den << 63
    Big sh = den;
    big_shl(sh, 63);
    unsigned long long q = 0;
    for (int b = 63; b >= 0; --b) {
        if (big_cmp(num, sh) >= 0) {
            big_sub(num, sh);
            q |= 1ull << b;
        }
        big_shr1(sh);
    }
    // num = remainder < den; compare 2*rem with den
    big_shl(num, 1);
    const int c = big_cmp(num, den);
    *up = c > 0 || (c == 0 && (q & 1ull));
    return q;
}

}  // namespace

__host__ __device__ int format_g17_f64(double v, char* out) {
    unsigned long long bits;
    memcpy(&bits, &v, 8);
    int o = 0;
    if (bits >> 63) out[o++] = '-';
    const unsigned ex = (unsigned)(bits >> 52) & 0x7ffu;
    const unsigned long long man = bits & 0xfffffffffffffull;
    if (ex == 0x7ffu) {
        const char* w = man ? "nan" : "inf";
        for (int i = 0; i < 3; ++i) out[o++] = w[i];
        return o;
    }
    if (ex == 0 && man == 0) {
        out[o++] = '0';
        return o;
    }
    const unsigned long long M = ex ? (man | (1ull << 52)) : man;
    const int E = ex ? (int)ex - 1075 : -1074;
    // X = floor(log10 v) exactly: the estimate is fixed on the TRUNCATED
    // 17-digit quotient (a double can sit within half a unit of 10^X, where the
    // rounded one would mislead); then the rounding may carry into 10^17.
    int X = (int)floor(log10((double)M) + E * 0.30102999566398120);
    unsigned long long D = 0;
    for (int guard = 0; guard < 4; ++guard) {
        bool up = false;
        D = scaled_floor64(M, E, 16 - X, &up);
        if (D >= 100000000000000000ull) {
            ++X;
        } else if (D < 10000000000000000ull) {
            --X;
        } else {
            D += up ? 1ull : 0ull;
            if (D == 100000000000000000ull) D = 10000000000000000ull, ++X;
            break;
        }
    }
    char dg[17];
    for (int i = 16; i >= 0; --i) {
        dg[i] = (char)('0' + (int)(D % 10ull));
        D /= 10ull;
    }
    int last = 16;
    while (last > 0 && dg[last] == '0') --last;
    if (X >= -4 && X < 17) {
        if (X >= 0) {
            for (int i = 0; i <= X; ++i) out[o++] = dg[i];
            if (last > X) {
                out[o++] = '.';
                for (int i = X + 1; i <= last; ++i) out[o++] = dg[i];
            }
        } else {
            out[o++] = '0';
            out[o++] = '.';
            for (int i = 0; i < -X - 1; ++i) out[o++] = '0';
            for (int i = 0; i <= last; ++i) out[o++] = dg[i];
        }
    } else {
        out[o++] = dg[0];
        if (last > 0) {
            out[o++] = '.';
            for (int i = 1; i <= last; ++i) out[o++] = dg[i];
        }
        out[o++] = 'e';
        out[o++] = X < 0 ? '-' : '+';
        const int ax = X < 0 ? -X : X;
        if (ax >= 100) out[o++] = (char)('0' + ax / 100);
        out[o++] = (char)('0' + (ax / 10) % 10);
        out[o++] = (char)('0' + ax % 10);
    }
    return o;
}

namespace {

__device__ __forceinline__ int format_u64(unsigned long long v, char* out) {
    char tmp[20];
    int n = 0;
    do {
        tmp[n++] = (char)('0' + (int)(v % 10ull));
        v /= 10ull;
    } while (v);
    for (int i = 0; i < n; ++i) out[i] = tmp[n - 1 - i];
    return n;
}

__device__ __forceinline__ int digits_u64(unsigned long long v) {
    int n = 1;
    while (v >= 10ull) v /= 10ull, ++n;
    return n;
}

// "%.17g" of entry e: the exact fp64 value when the handle keeps one.
__device__ __forceinline__ int format_entry(const float* vals, const double* vals64, int e, char* out) {
    return vals64 ? format_g17_f64(vals64[e], out) : format_g17(vals[e], out);
}

// Bytes of one entry line "r c v\n".
__device__ __forceinline__ int line_bytes(int row, int col, const float* vals, const double* vals64, int e) {
    char tmp[32];
    return digits_u64((unsigned long long)row + 1) + digits_u64((unsigned long long)col + 1) +
           format_entry(vals, vals64, e, tmp) + 3;
}

constexpr int kRowsPerBlock = 64;
constexpr int kStageBytes = 96 * 1024;

// Pass 1: bytes of each block of kRowsPerBlock rows.
__global__ void __launch_bounds__(256) text_size_kernel(const int32_t* row_ptr, const int32_t* col_idx,
                                                        const float* vals, const double* vals64, int rows,
                                                        unsigned long long* block_bytes) {
    __shared__ unsigned long long s_sum;
    if (threadIdx.x == 0) s_sum = 0;
    __syncthreads();
    const int r0 = blockIdx.x * kRowsPerBlock;
    const int r1 = min(rows, r0 + kRowsPerBlock);
    const int e0 = row_ptr[r0], e1 = row_ptr[r1];
    unsigned long long local = 0;
    // entries of the block, one thread per entry (row found by a short scan)
    int r = r0;
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        while (row_ptr[r + 1] <= e) ++r;
        local += (unsigned long long)line_bytes(r, col_idx[e], vals, vals64, e);
    }
    atomicAdd(&s_sum, local);
    __syncthreads();
    if (threadIdx.x == 0) block_bytes[blockIdx.x] = s_sum;
}

// Exclusive scan of the block totals in one CTA (blocks <= a few 10^5).
__global__ void __launch_bounds__(1024) text_scan_kernel(unsigned long long* v, int n,
                                                         unsigned long long base) {
    __shared__ unsigned long long s[1024];
    const int t = threadIdx.x;
    const int per = (n + 1023) / 1024;
    const int i0 = t * per, i1 = min(n, i0 + per);
    unsigned long long acc = 0;
    for (int i = i0; i < i1; ++i) acc += v[i];
    s[t] = acc;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const unsigned long long a = t >= o ? s[t - o] : 0;
        __syncthreads();
        s[t] += a;
        __syncthreads();
    }
    unsigned long long run = base + (t ? s[t - 1] : 0);
    for (int i = i0; i < i1; ++i) {
        const unsigned long long x = v[i];
        v[i] = run;
        run += x;
    }
    if (t == 1023) v[n] = base + s[1023];
}

// Pass 2: render each block's lines into shared memory, then copy out.
__global__ void __launch_bounds__(256) text_write_kernel(const int32_t* row_ptr, const int32_t* col_idx,
                                                         const float* vals, const double* vals64, int rows,
                                                         const unsigned long long* block_off,
                                                         char* out, int swap) {
    extern __shared__ unsigned char s_text[];
    __shared__ int s_lineoff[257];
    const int r0 = blockIdx.x * kRowsPerBlock;
    const int r1 = min(rows, r0 + kRowsPerBlock);
    const int e0 = row_ptr[r0], e1 = row_ptr[r1];
    const unsigned long long gbase = block_off[blockIdx.x];
    const unsigned long long total = block_off[blockIdx.x + 1] - gbase;
    // Entries in chunks of 256: per-entry line length -> block scan -> render.
    unsigned long long done = 0;  // bytes of this block already flushed
    int staged = 0;               // bytes currently in s_text
    int r = r0;
    for (int c0 = e0; c0 < e1; c0 += blockDim.x) {
        const int e = c0 + threadIdx.x;
        char line[64];
        int len = 0;
        if (e < e1) {
            while (row_ptr[r + 1] <= e) ++r;
            // CSR: "major minor"; CSC storage order prints (row = minor, col = major)
            const unsigned long long a = (unsigned long long)(swap ? col_idx[e] : r) + 1;
            const unsigned long long b = (unsigned long long)(swap ? r : col_idx[e]) + 1;
            len = format_u64(a, line);
            line[len++] = ' ';
            len += format_u64(b, line + len);
            line[len++] = ' ';
            len += format_entry(vals, vals64, e, line + len);
            line[len++] = '\n';
        }
        // exclusive scan of len over the CTA
        if (threadIdx.x == 0) s_lineoff[0] = 0;
        __syncthreads();
        s_lineoff[threadIdx.x + 1] = len;
        __syncthreads();
        for (int o = 1; o < 256; o <<= 1) {
            const int a = threadIdx.x + 1 > o ? s_lineoff[threadIdx.x + 1 - o] : 0;
            __syncthreads();
            s_lineoff[threadIdx.x + 1] += a;
            __syncthreads();
        }
        const int chunk = s_lineoff[256];
        if (staged + chunk > kStageBytes) {  // flush (the CTA's bytes are contiguous in `out`)
            for (int i = threadIdx.x; i < staged; i += blockDim.x) out[gbase + done + i] = s_text[i];
            done += staged;
            staged = 0;
            __syncthreads();
        }
        const int off = staged + s_lineoff[threadIdx.x];
        for (int i = 0; i < len; ++i) s_text[off + i] = line[i];
        staged += chunk;
        __syncthreads();
    }
    for (int i = threadIdx.x; i < staged; i += blockDim.x) out[gbase + done + i] = s_text[i];
    (void)total;
}

std::once_flag g_pow5_once[64];
cudaError_t g_pow5_err[64];

cudaError_t init_pow5(int dev) {
    std::call_once(g_pow5_once[dev & 63], [dev] {
        unsigned long long t[62][3];
        unsigned long long w[3] = {1, 0, 0};
        for (int k = 0; k < 62; ++k) {
            t[k][0] = w[0];
            t[k][1] = w[1];
            t[k][2] = w[2];
            unsigned __int128 c = 0;
            for (int i = 0; i < 3; ++i) {
                c += (unsigned __int128)w[i] * 5u;
                w[i] = (unsigned long long)c;
                c >>= 64;
            }
        }
        g_pow5_err[dev & 63] = cudaMemcpyToSymbol(c_pow5, t, sizeof t);
    });
    return g_pow5_err[dev & 63];
}

}  // namespace

// Renders the entry lines of a compressed matrix (device arrays, `rows` = its
// major dimension) into `out_dev` starting at byte `base`, in storage order
// (SparseMatrix::entries, inc/sparse.hpp:133-149); `swap` prints the minor
// index first (CSC: "row col" = "minor major").  The line length is symmetric
// in the two indices, so the size pass needs no flag.
// `scratch` holds (rows / 64 + 2) unsigned long longs.
cudaError_t render_entries(const int32_t* row_ptr, const int32_t* col_idx, const float* vals,
                           const double* vals64, int rows, unsigned long long* scratch, char* out_dev, unsigned long long base,
                           cudaStream_t st, bool size_only, bool swap) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t e = init_pow5(dev);
    if (e != cudaSuccess) return e;
    const int blocks = (rows + kRowsPerBlock - 1) / kRowsPerBlock;
    text_size_kernel<<<blocks, 256, 0, st>>>(row_ptr, col_idx, vals, vals64, rows, scratch);
    text_scan_kernel<<<1, 1024, 0, st>>>(scratch, blocks, base);
    if (size_only) return cudaGetLastError();
    static std::atomic<bool> attr[64];  // per device (benign concurrent first use)
    if (!attr[dev & 63]) {
        e = cudaFuncSetAttribute(text_write_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kStageBytes + 256 * 64);
        if (e != cudaSuccess) return e;
        attr[dev & 63] = true;
    }
    text_write_kernel<<<blocks, 256, kStageBytes + 256 * 64, st>>>(row_ptr, col_idx, vals, vals64, rows, scratch,
                                                                  out_dev, swap ? 1 : 0);
    return cudaGetLastError();
}

int text_rows_per_block() { return kRowsPerBlock; }

}  // namespace spb

extern "C" int spconv_format_g17(double v, char* out) {
    if (!out) return -1;
    const int n = spb::format_g17_f64(v, out);
    out[n] = '\0';
    return n;
}
