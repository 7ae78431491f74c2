/*
 * spconv_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C CPU restatement of the reference's conv-as-SpMV path
 * (/root/reference/proj/include/spconv, abbreviated `inc/` below).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path
 * (paper_2411_19419_b200/libspconv_b200.so) never links or calls it.
 *
 * Parity of this restatement is PINNED two ways (see tests/test_oracle.py):
 *   1. against oracle/_ref/libspconv_ref.so, the reference headers themselves
 *      compiled by oracle/Makefile (when /root/reference is present), and
 *   2. against the committed golden fixtures in tests/golden/, which were
 *      produced by that same compiled reference (tests/golden/make_golden.py).
 *
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction: the reference's
 * Release flags produce separate mul+add, inc/sparse.hpp:185-191).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* RNG: inc/rng.hpp                                                          */
/* ------------------------------------------------------------------------ */

/* inc/rng.hpp:19-25 */
uint64_t orc_splitmix64_next(uint64_t *state) {
    *state += 0x9E3779B97F4A7C15ull;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

typedef struct {
    uint64_t s[4];
    int has_spare;
    double spare;
} orc_normal;

/* inc/rng.hpp:29-31 (seeding), :53-55 (sampler state) */
static void normal_init(orc_normal *g, uint64_t seed) {
    for (int i = 0; i < 4; ++i) g->s[i] = orc_splitmix64_next(&seed);
    g->has_spare = 0;
    g->spare = 0.0;
}

/* inc/rng.hpp:33-44 (xoshiro256++) */
static uint64_t xoshiro_next(orc_normal *g) {
    uint64_t *s = g->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

/* inc/rng.hpp:47 */
static double uniform01(orc_normal *g) { return (double)(xoshiro_next(g) >> 11) * 0x1.0p-53; }

/* inc/rng.hpp:57-72 (Marsaglia polar method, spare returned second) */
static double normal_next(orc_normal *g) {
    if (g->has_spare) {
        g->has_spare = 0;
        return g->spare;
    }
    double u, v, s;
    do {
        u = 2.0 * uniform01(g) - 1.0;
        v = 2.0 * uniform01(g) - 1.0;
        s = u * u + v * v;
    } while (s >= 1.0 || s == 0.0);
    const double f = sqrt(-2.0 * log(s) / s);
    g->spare = v * f;
    g->has_spare = 1;
    return u * f;
}

/* random_normal_grid / random_normal_kernel fill order: inc/rng.hpp:80-92 */
void orc_random_normal(uint64_t seed, int64_t count, double *out) {
    orc_normal g;
    normal_init(&g, seed);
    for (int64_t i = 0; i < count; ++i) out[i] = normal_next(&g);
}

/* Same stream, rounded to fp32 (the parity recipe of SURVEY.md section 8c). */
void orc_random_normal_f32(uint64_t seed, int64_t count, float *out) {
    orc_normal g;
    normal_init(&g, seed);
    for (int64_t i = 0; i < count; ++i) out[i] = (float)normal_next(&g);
}

/* inc/rng.hpp:95-98 */
uint64_t orc_derive_seed(uint64_t base, uint64_t index) {
    uint64_t state = base ^ (0x9E3779B97F4A7C15ull * (index + 1));
    return orc_splitmix64_next(&state);
}

/* ------------------------------------------------------------------------ */
/* Geometry: inc/conv.hpp:33-62                                              */
/* ------------------------------------------------------------------------ */

/* inc/conv.hpp:42-47.  Returns 0 if valid, 1 on the first failing check,
 * 2 on the second (the reference's two std::invalid_argument messages). */
int orc_spec_check(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p) {
    if (m < 1 || n < 1 || k < 1 || s < 1 || p < 0) return 1;
    if (k > m + 2 * p || k > n + 2 * p) return 2;
    return 0;
}

/* inc/conv.hpp:52-53 */
int64_t orc_m_out(int64_t m, int64_t k, int64_t s, int64_t p) { return (m + 2 * p - k) / s + 1; }

static inline int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
static inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

/* ------------------------------------------------------------------------ */
/* Closed-form count: inc/analysis.hpp                                       */
/* ------------------------------------------------------------------------ */

/* inc/analysis.hpp:21-28 (c1) and :31-38 (c2) share this form. */
static int64_t c_pad(int64_t x, int64_t dim, int64_t k, int64_t s, int64_t p) {
    return max64(0, p - s * x) + max64(0, s * x + k - dim - p);
}

/* inc/analysis.hpp:42-52: max(0,k-c1(x))*max(0,k-c2(y)), raster order. */
void orc_nnz_per_output(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int64_t *out) {
    const int64_t mo = orc_m_out(m, k, s, p), no = orc_m_out(n, k, s, p);
    int64_t r = 0;
    for (int64_t x = 0; x < mo; ++x) {
        const int64_t rows = max64(0, k - c_pad(x, m, k, s, p));
        for (int64_t y = 0; y < no; ++y) out[r++] = rows * max64(0, k - c_pad(y, n, k, s, p));
    }
}

/* inc/analysis.hpp:56-66 */
int64_t orc_nnz_bound(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p) {
    const int64_t mo = orc_m_out(m, k, s, p), no = orc_m_out(n, k, s, p);
    int64_t total = 0;
    for (int64_t x = 0; x < mo; ++x) {
        const int64_t rows = max64(0, k - c_pad(x, m, k, s, p));
        for (int64_t y = 0; y < no; ++y) total += rows * max64(0, k - c_pad(y, n, k, s, p));
    }
    return total;
}

/* inc/analysis.hpp:70-89: brute-force mask overlap. */
int64_t orc_nnz_oracle(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p) {
    const int64_t pr = m + 2 * p, pc = n + 2 * p;
    char *mask = (char *)calloc((size_t)(pr * pc), 1);
    if (!mask) return -1;
    for (int64_t r = 0; r < m; ++r)
        for (int64_t c = 0; c < n; ++c) mask[(r + p) * pc + c + p] = 1;
    const int64_t mo = orc_m_out(m, k, s, p), no = orc_m_out(n, k, s, p);
    int64_t total = 0;
    for (int64_t x = 0; x < mo; ++x)
        for (int64_t y = 0; y < no; ++y)
            for (int64_t j = 0; j < k; ++j) {
                const int64_t base = (s * x + j) * pc + s * y;
                for (int64_t i = 0; i < k; ++i) total += mask[base + i];
            }
    free(mask);
    return total;
}

/* ------------------------------------------------------------------------ */
/* Transform T = C*P: inc/conv.hpp:125-204                                   */
/* ------------------------------------------------------------------------ */

/*
 * Restates build_transform (inc/conv.hpp:179-204).  The ColumnGather route
 * (:188-203) is followed literally: enumerate C's entries in CSR order
 * (row x*n_out+y, then padded column (s*x+j)*(n+2p)+s*y+i ascending, i.e.
 * (j,i) order, inc/conv.hpp:150-160), map each padded column through the
 * selector P (inc/conv.hpp:125-135) and keep it iff it lands inside the input
 * and the tap is != 0.0 (:201).  The Spgemm route (:182-186, the default)
 * produces acc = 0.0 + K*1.0 == K for every surviving (row, col) and drops
 * acc == 0.0 (inc/sparse.hpp:331-335), hence the identical result -- the
 * pinning tests check both routes of the real reference against this.
 * compile()'s sort (inc/sparse.hpp:93-97) is the identity here because the
 * enumeration is already (row, col)-ascending and the padded->input map is
 * monotone; no duplicate can arise (each (j,i) maps to a distinct column).
 *
 * Two-call protocol: pass ptr/idx/val == NULL to get nnz only.
 * Returns nnz, or -1 on an invalid spec.
 */
int64_t orc_build_transform(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p,
                            const double *kern, int64_t *ptr, int64_t *idx, double *val) {
    if (orc_spec_check(m, n, k, s, p) != 0) return -1;
    const int64_t mo = orc_m_out(m, k, s, p), no = orc_m_out(n, k, s, p);
    int64_t e = 0;
    if (ptr) ptr[0] = 0;
    for (int64_t x = 0; x < mo; ++x) {
        for (int64_t y = 0; y < no; ++y) {
            for (int64_t j = 0; j < k; ++j) {
                const int64_t pr = s * x + j; /* padded row */
                for (int64_t i = 0; i < k; ++i) {
                    const int64_t pc = s * y + i; /* padded col */
                    const double v = kern[j * k + i];
                    const int inside = pr >= p && pr < p + m && pc >= p && pc < p + n;
                    if (inside && v != 0.0) {
                        if (idx) {
                            idx[e] = (pr - p) * n + (pc - p);
                            val[e] = v;
                        }
                        ++e;
                    }
                }
            }
            if (ptr) ptr[x * no + y + 1] = e;
        }
    }
    return e;
}

/* The same enumeration written straight into the DEVICE format (int32
 * row_ptr / col_idx, fp32 vals) for full-size parity checks (205 M entries at
 * config 4) without the int64/f64 widening.  Returns nnz or -1. */
int64_t orc_build_transform_native(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p,
                                   const float *kern, int32_t *ptr, int32_t *idx, float *val) {
    if (orc_spec_check(m, n, k, s, p) != 0) return -1;
    const int64_t mo = orc_m_out(m, k, s, p), no = orc_m_out(n, k, s, p);
    int64_t e = 0;
    if (ptr) ptr[0] = 0;
    for (int64_t x = 0; x < mo; ++x)
        for (int64_t y = 0; y < no; ++y) {
            for (int64_t j = 0; j < k; ++j) {
                const int64_t pr = s * x + j;
                if (pr < p || pr >= p + m) continue;
                for (int64_t i = 0; i < k; ++i) {
                    const int64_t pc = s * y + i;
                    const float v = kern[j * k + i];
                    if (pc >= p && pc < p + n && v != 0.0f) {
                        if (idx) {
                            idx[e] = (int32_t)((pr - p) * n + (pc - p));
                            val[e] = v;
                        }
                        ++e;
                    }
                }
            }
            if (ptr) ptr[x * no + y + 1] = (int32_t)e;
        }
    return e;
}

/* fp32 ordered-fmaf SpMV over the native format (see orc_spmv_csr_f32_fma). */
void orc_spmm_native_f32_fma(int64_t rows, const int32_t *ptr, const int32_t *idx, const float *val,
                             const float *X, int64_t ldx, float *Y, int64_t ldy, int64_t batch) {
    for (int64_t b = 0; b < batch; ++b) {
        const float *x = X + b * ldx;
        float *y = Y + b * ldy;
        for (int64_t i = 0; i < rows; ++i) {
            float acc = 0.0f;
            for (int32_t e = ptr[i]; e < ptr[i + 1]; ++e) acc = fmaf(val[e], x[idx[e]], acc);
            y[i] = acc;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* SpMV: inc/sparse.hpp:180-192 (detail::spmv_csr_rows)                     */
/* ------------------------------------------------------------------------ */

/* fp64, column-ascending, separate multiply and add (no FMA) exactly as the
 * reference's Release build evaluates acc += val[k]*x[idx[k]]. */
void orc_spmv_csr_f64(int64_t rows, const int64_t *ptr, const int64_t *idx, const double *val,
                      const double *x, double *y) {
    for (int64_t i = 0; i < rows; ++i) {
        double acc = 0.0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
            const double prod = val[k] * x[idx[k]];
            acc = acc + prod;
        }
        y[i] = acc;
    }
}

/* The fp32 contract of the device path: the same loop in fp32 with one
 * rounding per step via fmaf (acc = fmaf(val, x, acc)), starting from +0.0f.
 * The device kernels accumulate each row in exactly this order, so their
 * output is expected to be BIT-identical to this function. */
void orc_spmv_csr_f32_fma(int64_t rows, const int64_t *ptr, const int64_t *idx, const float *val,
                          const float *x, float *y) {
    for (int64_t i = 0; i < rows; ++i) {
        float acc = 0.0f;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) acc = fmaf(val[k], x[idx[k]], acc);
        y[i] = acc;
    }
}

/* Batched form of the above over image-major X[b*ldx + col] -> Y[b*ldy + row]. */
void orc_spmm_csr_f32_fma(int64_t rows, const int64_t *ptr, const int64_t *idx, const float *val,
                          const float *X, int64_t ldx, float *Y, int64_t ldy, int64_t batch) {
    for (int64_t b = 0; b < batch; ++b)
        orc_spmv_csr_f32_fma(rows, ptr, idx, val, X + b * ldx, Y + b * ldy);
}

/* Condition number of each output, sum_e |val_e * x_col_e|, for the
 * condition-aware tolerance |y_gpu - y_ref| <= tol * cond. */
void orc_spmv_abs_f64(int64_t rows, const int64_t *ptr, const int64_t *idx, const double *val,
                      const double *x, double *cond) {
    for (int64_t i = 0; i < rows; ++i) {
        double acc = 0.0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) acc += fabs(val[k] * x[idx[k]]);
        cond[i] = acc;
    }
}

/* ------------------------------------------------------------------------ */
/* Direct sliding window: inc/reference.hpp:41-61 (secondary oracle)         */
/* ------------------------------------------------------------------------ */
int orc_direct_conv(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, const double *a,
                    const double *kern, double *out) {
    if (orc_spec_check(m, n, k, s, p) != 0) return 1;
    const int64_t mo = orc_m_out(m, k, s, p), no = orc_m_out(n, k, s, p);
    for (int64_t x = 0; x < mo; ++x)
        for (int64_t y = 0; y < no; ++y) {
            double acc = 0.0;
            for (int64_t j = 0; j < k; ++j)
                for (int64_t i = 0; i < k; ++i) {
                    const int64_t r = s * x + j - p, c = s * y + i - p;
                    const double a_v = (r >= 0 && r < m && c >= 0 && c < n) ? a[r * n + c] : 0.0;
                    const double prod = kern[j * k + i] * a_v;
                    acc = acc + prod;
                }
            out[x * no + y] = acc;
        }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* CSC layout: relayout (inc/sparse.hpp:268-274) and CSC SpMV (:194-205)     */
/* ------------------------------------------------------------------------ */

/* relayout(m, other) re-compiles m's entries in the other layout
 * (SparseMatrix::compile, inc/sparse.hpp:85-119: sort by (major, minor),
 * histogram, prefix).  For a valid matrix that is a stable transposition of
 * the storage: optr[c] = #entries with minor < c, and visiting the majors in
 * ascending order fills every output slice in ascending (new minor) order --
 * a counting sort, no comparison sort needed.  `major` / `minor` are the
 * input's major and minor dimensions; optr has minor+1 entries. */
void orc_transpose(int64_t major, int64_t minor, const int64_t *ptr, const int64_t *idx,
                   const double *val, int64_t *optr, int64_t *oidx, double *oval) {
    for (int64_t c = 0; c <= minor; ++c) optr[c] = 0;
    for (int64_t e = 0; e < ptr[major]; ++e) optr[idx[e] + 1]++;
    for (int64_t c = 0; c < minor; ++c) optr[c + 1] += optr[c];
    int64_t *cur = (int64_t *)malloc((size_t)(minor > 0 ? minor : 1) * sizeof(int64_t));
    for (int64_t c = 0; c < minor; ++c) cur[c] = optr[c];
    for (int64_t r = 0; r < major; ++r)
        for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
            const int64_t q = cur[idx[e]]++;
            oidx[q] = r;
            oval[q] = val[e];
        }
    free(cur);
}

/* detail::spmv_csc_cols (inc/sparse.hpp:194-205) on one thread (spmv's nt <= 1
 * branch, :227-231): y = 0; for every column j ascending, y[idx] += val * x[j]
 * (fp64, separate multiply and add).  Every output therefore sums its terms
 * in column-ascending order from +0.0, exactly as spmv_csr_rows does. */
void orc_spmv_csc_f64(int64_t cols, const int64_t *ptr, const int64_t *idx, const double *val,
                      const double *x, double *y, int64_t rows) {
    for (int64_t i = 0; i < rows; ++i) y[i] = 0.0;
    for (int64_t j = 0; j < cols; ++j) {
        const double xj = x[j];
        for (int64_t k = ptr[j]; k < ptr[j + 1]; ++k) {
            const double prod = val[k] * xj;
            y[idx[k]] = y[idx[k]] + prod;
        }
    }
}

/* spmv with nt > 1 threads on a CSC matrix (inc/sparse.hpp:221-258): nt is
 * capped at the column count, columns are cut into chunks of ceil(cols / nt),
 * thread t scatters chunk t into its own partial vector (from 0.0), and the
 * partials are added to y (from 0.0) in thread order. */
void orc_spmv_csc_f64_threads(int64_t cols, const int64_t *ptr, const int64_t *idx, const double *val,
                              const double *x, double *y, int64_t rows, int64_t nt) {
    if (nt > cols) nt = cols > 0 ? cols : 1;
    if (nt <= 1) {
        orc_spmv_csc_f64(cols, ptr, idx, val, x, y, rows);
        return;
    }
    const int64_t chunk = (cols + nt - 1) / nt;
    double *part = (double *)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1));
    for (int64_t i = 0; i < rows; ++i) y[i] = 0.0;
    for (int64_t t = 0; t < nt; ++t) {
        int64_t lo = t * chunk < cols ? t * chunk : cols;
        int64_t hi = lo + chunk < cols ? lo + chunk : cols;
        for (int64_t i = 0; i < rows; ++i) part[i] = 0.0;
        for (int64_t j = lo; j < hi; ++j) {
            const double xj = x[j];
            for (int64_t k = ptr[j]; k < ptr[j + 1]; ++k) {
                const double prod = val[k] * xj;
                part[idx[k]] = part[idx[k]] + prod;
            }
        }
        for (int64_t i = 0; i < rows; ++i) y[i] = y[i] + part[i];
    }
    free(part);
}

/* The same scatter in fp32 with one rounding per step (fmaf): the device
 * contract for CSC transforms.  Per output it is the CSR ordered-fmaf chain,
 * so it is bit-identical to orc_spmv_csr_f32_fma on the transposed storage. */
void orc_spmv_csc_f32_fma(int64_t cols, const int64_t *ptr, const int64_t *idx, const float *val,
                          const float *x, float *y, int64_t rows) {
    for (int64_t i = 0; i < rows; ++i) y[i] = 0.0f;
    for (int64_t j = 0; j < cols; ++j) {
        const float xj = x[j];
        for (int64_t k = ptr[j]; k < ptr[j + 1]; ++k) y[idx[k]] = fmaf(val[k], xj, y[idx[k]]);
    }
}
