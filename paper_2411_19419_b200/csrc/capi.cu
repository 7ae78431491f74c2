// capi.cu -- the extern "C" boundary declared in include/spconv_b200.h.
//
// Host-side orchestration only: argument validation with the reference's
// exception messages, the O(k^2 + m_out + n_out) host tables of the closed-form
// CSR build, kernel-path selection (run_spmm), the chunked host<->device
// pipeline of spconv_convolve_host, and the text parsing of read_transform /
// read_sparse.  All arithmetic on T and on images happens in the CUDA kernels
// of csr_build.cu, csc_build.cu, spmm.cu, spmm_band.cu, text_io.cu and
// verify.cu; there is no CPU fallback.  (Matrices that arrive from the host --
// uploads and non-conv text files -- are transposed on the host for relayout.)
#include <cudaTypedefs.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/spconv_b200.h"
#include "internal.h"

using spb::Geom;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(SPCONV_ECUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                                  cudaGetErrorString(e) + ")");
}

#define CK(call)                                              \
    do {                                                      \
        cudaError_t e_ = (call);                              \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
    } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

std::string spec_str(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "(m=%lld, n=%lld, k=%lld, s=%lld, p=%lld)", (long long)m,
                  (long long)n, (long long)k, (long long)s, (long long)p);
    return buf;
}

// inc/conv.hpp:42-47 (same messages).
int check_spec(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p) {
    if (m < 1 || n < 1 || k < 1 || s < 1 || p < 0)
        return fail(SPCONV_EINVAL,
                    "ConvSpec: need m,n,k,s >= 1 and p >= 0, got " + spec_str(m, n, k, s, p));
    if (k > m + 2 * p || k > n + 2 * p)
        return fail(SPCONV_EINVAL, "ConvSpec: kernel larger than padded input, " +
                                       spec_str(m, n, k, s, p));
    return SPCONV_OK;
}

Geom make_geom(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p) {
    Geom g{m, n, k, s, p, (m + 2 * p - k) / s + 1, (n + 2 * p - k) / s + 1};
    return g;
}

// Valid tap range along one axis (see csr_build.cu).
inline void tap_range(int64_t x, int64_t dim, int64_t k, int64_t s, int64_t p, int64_t& lo,
                      int64_t& hi) {
    lo = std::max<int64_t>(0, p - s * x);
    hi = std::min<int64_t>(k, dim + p - s * x);
    lo = std::min(lo, k);
    if (hi < lo) hi = lo;
}

// Host tables of the closed-form build: O(k^2 + m_out + n_out) work.
struct HostTables {
    std::vector<float> taps;
    std::vector<int32_t> sat;
    std::vector<long long> w;  // W[j] = sum_i nz[j][i] * #{y : i in I(y)}
    int64_t nnz = 0;
    int64_t k2max = 0;
    bool dense = true;    // every tap non-zero and finite
    bool nonzero = true;  // every tap non-zero
};

void make_tables(const Geom& g, const float* kernel, HostTables& ht) {
    const int64_t k = g.k, k1 = k + 1;
    ht.taps.assign(kernel, kernel + k * k);
    ht.sat.assign((size_t)(k1 * k1), 0);
    ht.dense = true;
    ht.nonzero = true;
    for (int64_t q = 0; q < k * k; ++q) {
        ht.dense &= kernel[q] != 0.0f && std::isfinite(kernel[q]);
        ht.nonzero &= kernel[q] != 0.0f;
    }
    for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i < k; ++i)
            ht.sat[(j + 1) * k1 + i + 1] = ht.sat[j * k1 + i + 1] + ht.sat[(j + 1) * k1 + i] -
                                           ht.sat[j * k1 + i] + (kernel[j * k + i] != 0.0f ? 1 : 0);
    auto rect = [&](int64_t jlo, int64_t jhi, int64_t ilo, int64_t ihi) -> int64_t {
        return ht.sat[jhi * k1 + ihi] - ht.sat[jlo * k1 + ihi] - ht.sat[jhi * k1 + ilo] +
               ht.sat[jlo * k1 + ilo];
    };
    // cntY[i] = #{y : i in I(y)} via a difference array over the y-ranges.
    std::vector<int64_t> diff((size_t)k1, 0);
    std::vector<std::pair<int64_t, int64_t>> yr;  // distinct (ilo, ihi)
    for (int64_t y = 0; y < g.no; ++y) {
        int64_t lo, hi;
        tap_range(y, g.n, k, g.s, g.p, lo, hi);
        diff[lo] += 1;
        diff[hi] -= 1;
        if (yr.empty() || yr.back() != std::make_pair(lo, hi)) yr.emplace_back(lo, hi);
    }
    std::vector<int64_t> cnty((size_t)k, 0);
    int64_t run = 0;
    for (int64_t i = 0; i < k; ++i) cnty[i] = (run += diff[i]);
    // W[j]; RowTot(x) = sum_{j in J(x)} W[j].
    ht.w.assign((size_t)k, 0);
    std::vector<int64_t> pw((size_t)k1, 0);
    for (int64_t j = 0; j < k; ++j) {
        int64_t wj = 0;
        for (int64_t i = 0; i < k; ++i) wj += (kernel[j * k + i] != 0.0f ? 1 : 0) * cnty[i];
        ht.w[j] = wj;
        pw[j + 1] = pw[j] + wj;
    }
    std::sort(yr.begin(), yr.end());
    yr.erase(std::unique(yr.begin(), yr.end()), yr.end());
    ht.nnz = 0;
    ht.k2max = 0;
    std::pair<int64_t, int64_t> last_xr(-1, -1);
    for (int64_t x = 0; x < g.mo; ++x) {
        int64_t jlo, jhi;
        tap_range(x, g.m, k, g.s, g.p, jlo, jhi);
        ht.nnz += pw[jhi] - pw[jlo];
        if (std::make_pair(jlo, jhi) != last_xr) {
            last_xr = {jlo, jhi};
            for (auto& q : yr) ht.k2max = std::max(ht.k2max, rect(jlo, jhi, q.first, q.second));
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// Kernel-path selection (spconv_set_option "path"): auto (default) = the
// latency kernel for batch <= 2 (csr_spmv_bulk: closed-form row runs for
// conv transforms), else the band path (CSR band check + register-blocked
// apply) when instantiated for (k, s) with finite taps, else tiled (TMA when
// the strides allow); generic for uploaded matrices.  The forced values exist
// for cross-checking the paths.
enum Path { kAuto = 0, kBanded, kTiled, kTiledNoTma, kGeneric, kSpmv, kSpmvPlain };

Path path_override() { return static_cast<Path>(spb::opt(spb::kOptPath)); }

// 3-D tensor map over the batch X[b][m][n] (fp32) with the given box.
int encode_x_map(CUtensorMap* tmap, const void* X, const Geom& g, int64_t ldx, int64_t batch,
                 int box_c, int box_r, int box_b, bool f64 = false, int64_t row_pitch = 0) {
    std::memset(tmap, 0, sizeof *tmap);
    const int64_t es = f64 ? 8 : 4;
    const cuuint64_t dims[3] = {(cuuint64_t)g.n, (cuuint64_t)g.m, (cuuint64_t)batch};
    const cuuint64_t strides[2] = {(cuuint64_t)((row_pitch > 0 ? row_pitch : g.n) * es), (cuuint64_t)(ldx * es)};
    const cuuint32_t box[3] = {(cuuint32_t)box_c, (cuuint32_t)box_r, (cuuint32_t)box_b};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = encode_fn()(tmap, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                              const_cast<void*>(X), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS)
        return fail(SPCONV_ECUDA, "cuTensorMapEncodeTiled failed with CUresult " +
                                      std::to_string((int)cr));
    return SPCONV_OK;
}

// Band path over images whose rows TMA cannot describe (not 16-byte pitched,
// or a misaligned base): one coalesced pass copies them into 16-byte pitched
// rows (repitch.cu, a stream-ordered allocation freed once the launches are
// enqueued) and the tensor map describes the copy, so the windows are TMA
// boxes instead of element copies from one producer warp -- 1023^2 k3 at 64
// images 388 -> see DESIGN.  The per-entry fallback keeps reading X itself.
// Option repitch = off keeps the element staging.
struct RepitchBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    ~RepitchBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

int repitch_for_tma(const spconv_csr* h, const void* X, int64_t ldx, int64_t batch, bool f64, spb::BandParams& bp,
                    const spb::BandShape& sh, CUtensorMap* tmap, RepitchBuf& rb, cudaStream_t st) {
    const Geom& g = h->g;
    if (!bp.notma || spb::opt(spb::kOptRepitch) == 1 || encode_fn() == nullptr) return SPCONV_OK;
    if (g.m >= (1ll << 30) || g.n >= (1ll << 30)) return SPCONV_OK;
    const int64_t es = f64 ? 8 : 4, E = 16 / es;
    const int64_t np = (g.n + E - 1) / E * E;
    const double bytes = (double)batch * (double)g.m * (double)np * (double)es;
    if (bytes > 8.0 * (1ull << 30) || batch > 65535 || g.m * g.n > (1ll << 31))
        return SPCONV_OK;  // (a huge batch keeps the element staging)
    if (cudaMallocAsync(&rb.p, (size_t)bytes, st) != cudaSuccess) {  // (no room: keep the element staging)
        cudaGetLastError();
        rb.p = nullptr;
        return SPCONV_OK;
    }
    rb.st = st;
    CK(spb::launch_repitch(X, ldx, rb.p, (int)g.m, (int)g.n, np, batch, f64, st));
    if (int rc = encode_x_map(tmap, rb.p, g, g.m * np, batch, sh.wc, sh.wr, 1, f64, np)) return rc;
    bp.notma = 0;
    return SPCONV_OK;
}

// Transforms are allocated from the device's stream-ordered pool; keep freed
// blocks in the pool (instead of unmapping them at every synchronisation) so a
// rebuild costs the kernel, not a page-table update.
void keep_pool_memory(int device) {
    static std::once_flag flags[64];
    std::call_once(flags[device & 63], [device] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
}

int device_sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// ---- CSC conv transforms: verdict words, tap tables, the exposed-storage protocol ----

// One mapped (zero-copy) host word per CSC conv handle: device checks that
// fail store 1 there, and the next host call on the handle reads it without a
// synchronisation (a sticky verdict, like CUDA's sticky errors).
std::mutex g_flag_mu;
std::vector<int*> g_flag_free;

int* flag_alloc() {
    std::lock_guard<std::mutex> lk(g_flag_mu);
    if (g_flag_free.empty()) {
        int* page = nullptr;
        constexpr int kWords = 1024;  // one 4 KB page of words; never released
        if (cudaHostAlloc(reinterpret_cast<void**>(&page), kWords * sizeof(int),
                          cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
            return nullptr;
        for (int i = kWords - 1; i >= 0; --i) g_flag_free.push_back(page + i);
    }
    int* w = g_flag_free.back();
    g_flag_free.pop_back();
    *reinterpret_cast<volatile int*>(w) = 0;
    return w;
}

void flag_free(int* w) {
    if (!w) return;
    std::lock_guard<std::mutex> lk(g_flag_mu);
    g_flag_free.push_back(w);
}

bool csc_native(const spconv_csr* h) { return h->layout == 1 && h->is_conv && !h->row_ptr && h->csc_ptr; }

// Stored = the DOUBLE tap is non-zero when the handle keeps doubles (a tap that
// narrows to 0.0f is still an entry), else the fp32 tap (inc/sparse.hpp:335).
bool tap_stored(const spconv_csr* h, size_t q) {
    return h->host_taps64.empty() ? h->host_taps[q] != 0.0f : h->host_taps64[q] != 0.0;
}

// W[j] = sum over stored (j, i) of #{y : 0 <= s y + i - p < n} (the CSC column
// offsets' closed form; = sum_y cy(y) = sy for a kernel without zero taps).
void csc_tables(const spconv_csr* h, spb::CscGatherParams& cp) {
    const Geom& g = h->g;
    cp.zt = 0;
    for (int64_t j = 0; j < g.k && j < 32; ++j) {
        uint32_t row = 0;
        long long wj = 0;
        for (int64_t i = 0; i < g.k; ++i) {
            if (!tap_stored(h, (size_t)(j * g.k + i))) {
                cp.zt = 1;
                continue;
            }
            row |= 1u << i;
            const int64_t lo = g.p - i <= 0 ? 0 : (g.p - i + g.s - 1) / g.s;
            const int64_t hi = g.n + g.p - i - 1 < 0 ? -1 : std::min<int64_t>(g.no - 1, (g.n + g.p - i - 1) / g.s);
            wj += std::max<int64_t>(0, hi - lo + 1);
        }
        cp.nzrow[j] = row;
        cp.zw[j] = wj;
    }
}

spb::CscGatherParams csc_params(const spconv_csr* h, bool f64) {
    spb::CscGatherParams cp{};
    const Geom& g = h->g;
    cp.col_ptr = h->csc_ptr;
    cp.row_idx = h->csc_idx;
    cp.vals = h->csc_vals;
    cp.vals64 = f64 ? h->csc_vals64 : nullptr;
    cp.taps32 = h->taps;
    cp.taps64 = f64 ? h->taps64 : nullptr;
    cp.m = (int)g.m;
    cp.n = (int)g.n;
    cp.k = (int)g.k;
    cp.s = (int)g.s;
    cp.p = (int)g.p;
    cp.mo = (int)g.mo;
    cp.no = (int)g.no;
    cp.rows = h->rows;
    cp.cols = h->cols;
    cp.nnz = h->nnz;
    cp.fail = h->fail_flag;
    csc_tables(h, cp);
    if (g.k <= 7 && h->host_taps64.empty() && h->host_taps.size() == (size_t)(g.k * g.k)) {
        cp.inline_taps = 1;
        for (size_t q = 0; q < h->host_taps.size(); ++q) cp.it32[q] = h->host_taps[q];
    }
    return cp;
}

int csc_sticky(const spconv_csr* h, const char* who) {
    if (h->fail_flag && !h->exposed.load() && *reinterpret_cast<volatile int*>(h->fail_flag))
        return fail(SPCONV_ECUDA, std::string(who) +
                                      ": the stored matrix no longer matches the transform of its taps "
                                      "(a device check failed in an earlier call)");
    return SPCONV_OK;
}

// Exposed CSC handles (spconv_csr_device_ptrs handed out the arrays): the
// storage is checked on the device and the host waits for the verdict; when it
// no longer is the transform of the taps, the call applies the storage as it
// stands (repair_apply) -- the reference's scatter semantics.  Not capturable.
int band_setup(spconv_csr* h, bool csc, bool f64, int64_t batch, const void* X, int64_t ldx, void* Y, int64_t ldy,
               spb::BandParams& bp, spb::BandShape& sh, int sms, cudaStream_t st);
bool band_taps_ok(const spconv_csr* h);

int csc_exposed_clean(spconv_csr* h, cudaStream_t st, bool f64, bool* clean) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(st, &cap));
    if (cap != cudaStreamCaptureStatusNone)
        return fail(SPCONV_EINVAL, "a CSC handle whose arrays were handed out by spconv_csr_device_ptrs "
                                   "cannot be applied under stream capture");
    int* d = nullptr;
    CK(cudaMallocAsync(&d, sizeof(int), st));
    int v = 1;
    cudaError_t e = cudaMemsetAsync(d, 0, sizeof(int), st);
    const Geom& g = h->g;
    if (h->band_tw > 0 && h->csc_tiles_b > 0 && band_taps_ok(h) && spb::band_supported((int)g.k, (int)g.s)) {
        // band geometries: the CSC band check itself (segment by segment,
        // the kernel the batched apply runs), its verdict into d
        spb::BandParams bp{};
        spb::BandShape sh{};
        const int sms = device_sm_count();
        if (int rc = band_setup(h, true, false, 1, nullptr, 0, nullptr, 0, bp, sh, sms, st)) {
            cudaFreeAsync(d, st);
            return rc;
        }
        bp.fail_count = d;
        h->checked.store(true);
        if (e == cudaSuccess) e = spb::launch_band_check((int)g.k, (int)g.s, bp, st, sms);
    } else {
        spb::CscGatherParams cp = csc_params(h, f64);
        cp.fail = d;
        cp.verify_only = 1;
        if (e == cudaSuccess) e = spb::launch_csc_gather(cp, f64, st, device_sm_count());
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&v, d, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(d, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "CSC storage check");
    *clean = v == 0;
    return SPCONV_OK;
}

// y = the reference's CSC scatter over the storage as it stands (inc/sparse.hpp:
// 194-205, 243-258): entries in (column, position) order regrouped by row --
// a stable counting sort on the host -- then the row-major kernels (fp32
// ordered fmaf, or fp64 with the thread-chunk combine).
int csc_repair_apply(spconv_csr* h, const void* X, int64_t ldx, void* Y, int64_t ldy, int64_t batch,
                     cudaStream_t st, bool f64, int64_t chunk) {
    const int64_t rows = h->rows, cols = h->cols, nnz = h->nnz;
    std::vector<int32_t> cpv((size_t)cols + 1), ri((size_t)std::max<int64_t>(nnz, 1));
    std::vector<float> cv((size_t)std::max<int64_t>(nnz, 1));
    std::vector<double> cv64;
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(cpv.data(), h->csc_ptr, cpv.size() * 4, cudaMemcpyDeviceToHost));
    if (nnz > 0) {
        CK(cudaMemcpy(ri.data(), h->csc_idx, (size_t)nnz * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(cv.data(), h->csc_vals, (size_t)nnz * 4, cudaMemcpyDeviceToHost));
        if (f64 && h->csc_vals64) {
            cv64.resize((size_t)nnz);
            CK(cudaMemcpy(cv64.data(), h->csc_vals64, (size_t)nnz * 8, cudaMemcpyDeviceToHost));
        }
    }
    for (int64_t c = 0; c < cols; ++c)
        if (cpv[(size_t)c] < 0 || cpv[(size_t)c] > cpv[(size_t)c + 1] || cpv[(size_t)c + 1] > nnz)
            return fail(SPCONV_EINVAL, "CSC storage altered through spconv_csr_device_ptrs: col_ptr is not "
                                       "non-decreasing within [0, nnz]");
    std::vector<int32_t> rp((size_t)rows + 1, 0);
    int64_t used = 0;
    for (int64_t c = 0; c < cols; ++c)
        for (int32_t e = cpv[(size_t)c]; e < cpv[(size_t)c + 1]; ++e) {
            if (ri[(size_t)e] < 0 || ri[(size_t)e] >= rows)
                return fail(SPCONV_EINVAL, "CSC storage altered through spconv_csr_device_ptrs: row index " +
                                               std::to_string(ri[(size_t)e]) + " out of range");
            ++rp[(size_t)ri[(size_t)e] + 1];
            ++used;
        }
    for (int64_t r = 0; r < rows; ++r) rp[(size_t)r + 1] += rp[(size_t)r];
    std::vector<int32_t> cur(rp.begin(), rp.end() - 1), ci((size_t)std::max<int64_t>(used, 1));
    std::vector<float> vv((size_t)std::max<int64_t>(used, 1));
    std::vector<double> vv64(cv64.empty() ? 0 : (size_t)std::max<int64_t>(used, 1));
    for (int64_t c = 0; c < cols; ++c)
        for (int32_t e = cpv[(size_t)c]; e < cpv[(size_t)c + 1]; ++e) {
            const int32_t d = cur[(size_t)ri[(size_t)e]]++;
            ci[(size_t)d] = (int32_t)c;
            vv[(size_t)d] = cv[(size_t)e];
            if (!vv64.empty()) vv64[(size_t)d] = cv64[(size_t)e];
        }
    const size_t b_rp = ((rp.size() * 4) + 255) & ~size_t(255), b_ix = ((ci.size() * 4) + 255) & ~size_t(255);
    char* mem = nullptr;
    CK(cudaMalloc(&mem, b_rp + 2 * b_ix + vv64.size() * 8 + 256));
    auto* d_rp = reinterpret_cast<int32_t*>(mem);
    auto* d_ci = reinterpret_cast<int32_t*>(mem + b_rp);
    auto* d_vv = reinterpret_cast<float*>(mem + b_rp + b_ix);
    auto* d_v64 = vv64.empty() ? nullptr : reinterpret_cast<double*>(mem + b_rp + 2 * b_ix);
    cudaError_t e = cudaMemcpy(d_rp, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_ci, ci.data(), ci.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_vv, vv.data(), vv.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && d_v64) e = cudaMemcpy(d_v64, vv64.data(), vv64.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        if (f64) {
            spb::F64Params fp{d_rp, d_ci, d_vv, d_v64, static_cast<const double*>(X), ldx, static_cast<double*>(Y),
                              ldy, (int)rows, (int)batch};
            fp.chunk = chunk;
            e = spb::launch_spmm_f64(fp, st);
        } else {
            spb::GenericParams gp{d_rp, d_ci, d_vv, static_cast<const float*>(X), ldx, static_cast<float*>(Y), ldy,
                                  (int)rows, (int)batch};
            e = spb::launch_generic(gp, st);
        }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(mem);
    if (e != cudaSuccess) return cuda_fail(e, "CSC apply of the altered storage");
    return SPCONV_OK;
}

// The blocked apply needs finite taps; exact-zero taps (not stored) take the
// masked (ZT) instantiations: k <= 7, so the mask fits 64 bits.  (stored = the
// DOUBLE tap is non-zero when the handle has double taps: a tap that narrows
// to 0.0f is still an entry, applied as w = 0)
bool band_taps_ok(const spconv_csr* h) {
    bool finite = !h->host_taps.empty(), any = false;
    for (size_t q = 0; q < h->host_taps.size(); ++q) finite &= std::isfinite(h->host_taps[q]), any |= tap_stored(h, q);
    return h->taps_dense || (finite && any && h->g.k <= 7);
}

// BandParams of one band call (check + apply) over the handle's storage.
int band_setup(spconv_csr* h, bool csc, bool f64, int64_t batch, const void* X, int64_t ldx, void* Y, int64_t ldy,
               spb::BandParams& bp, spb::BandShape& sh, int sms, cudaStream_t st = nullptr) {
    const Geom& g = h->g;
    const bool band_taps = band_taps_ok(h);
    unsigned long long nzmask = 0;
    for (size_t q = 0; q < h->host_taps.size() && q < 64; ++q)
        if (tap_stored(h, q)) nzmask |= 1ull << q;
    bp = spb::BandParams{};
    bp.p = (int)g.p;
    bp.zt = band_taps && !h->taps_dense ? 1 : 0;
    bp.nzmask = nzmask;
    if (bp.zt) {  // W[j] = sum over stored taps (j, i) of #{y : tap i lands in the input}
        for (int64_t j = 0; j < g.k && j < 8; ++j) {
            long long wj = 0;
            for (int64_t i = 0; i < g.k; ++i) {
                if (!((nzmask >> (j * g.k + i)) & 1ull)) continue;
                // y with 0 <= s*y + i - p < n, y in [0, n_out): a closed range
                const int64_t lo = g.p - i <= 0 ? 0 : (g.p - i + g.s - 1) / g.s;
                const int64_t hi = g.n + g.p - i - 1 < 0 ? -1 : std::min<int64_t>(g.no - 1, (g.n + g.p - i - 1) / g.s);
                wj += std::max<int64_t>(0, hi - lo + 1);
            }
            bp.zw[j] = wj;
        }
    }
    CK(f64 ? spb::launch_band64((int)g.k, (int)g.s, bp, nullptr, st, &sh, sms)
           : spb::launch_band((int)g.k, (int)g.s, bp, nullptr, st, &sh, sms));
    bp.row_ptr = csc ? h->csc_ptr : h->row_ptr;
    bp.col_idx = csc ? h->csc_idx : h->col_idx;
    bp.vals = csc ? h->csc_vals : h->vals;
    bp.csc = csc ? 1 : 0;
    bp.tiles_b = h->csc_tiles_b;
    bp.fail_count = h->fail_flag;
    // Row-major storage handed out by spconv_csr_device_ptrs may change: the
    // fused form then recomputes failed segments (conv_band_fixup).  Otherwise
    // a failed check can only mean corrupted memory: it raises the verdict
    // word instead, and no fixup pass is launched.
    bp.fixup = !csc && h->exposed.load() ? 1 : 0;
    bp.taps = h->taps;
    bp.taps64 = f64 ? h->taps64 : nullptr;
    bp.vals64 = f64 ? h->vals64 : nullptr;
    bp.seg_ok = h->seg_ok;
    bp.X = static_cast<const float*>(X);
    bp.ldx = ldx;
    bp.Y = static_cast<float*>(Y);
    bp.ldy = ldy;
    bp.batch = (int)batch;
    bp.m = (int)g.m;
    bp.n = (int)g.n;
    bp.mo = (int)g.mo;
    bp.no = (int)g.no;
    bp.tiles_y = (int)((g.no + sh.tw - 1) / sh.tw);
    bp.tiles = (int)(((g.mo + sh.th - 1) / sh.th) * bp.tiles_y);
    bp.seg_div = spb::band_seg_div((int)g.k, (int)g.s);
    const int segw = sh.tw / bp.seg_div;
    bp.tiles_y_chk = (int)((g.no + segw - 1) / segw);
    // X rows TMA cannot describe (pitch not a multiple of 16 bytes, misaligned
    // base): the producer stages windows with cp.async element copies
    const int64_t eb = f64 ? 8 : 4;
    bp.notma = !((g.n * eb) % 16 == 0 && (ldx * eb) % 16 == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0 &&
                 encode_fn() != nullptr && g.m < (1ll << 30) && g.n < (1ll << 30)) ? 1 : 0;
    bp.fast_allowed = band_taps ? 1 : 0;
    bp.sy = (int)h->sy;
    bp.nnz = (int)h->nnz;
    const int cpt = sh.tw / 32, es = f64 ? 8 : 4;
    bp.y_vec = (ldy % cpt == 0) && (g.no % cpt == 0) && (reinterpret_cast<uintptr_t>(Y) % (es * cpt) == 0) &&
               (!f64 || reinterpret_cast<uintptr_t>(Y) % 16 == 0);
    return SPCONV_OK;
}

int run_spmm(spconv_csr* h, const float* X, int64_t ldx, float* Y, int64_t ldy,
             int64_t batch, cudaStream_t st) {
    if (batch == 0) return SPCONV_OK;
    if (batch > INT32_MAX) return fail(SPCONV_EINVAL, "spconv_spmm: batch exceeds int32");
    const Path force = path_override();
    const Geom& g = h->g;
    const bool tma_ok = h->is_conv && (g.n % 4 == 0) && (ldx % 4 == 0) &&
                        (reinterpret_cast<uintptr_t>(X) % 16 == 0) && encode_fn() != nullptr &&
                        g.m < (1ll << 30) && g.n < (1ll << 30);

    if (int rc = csc_sticky(h, "spconv_spmm")) return rc;
    // ---- CSC storage of a conv transform: the CSC kernels ----
    const bool csc = csc_native(h);
    if (csc) {
        if (h->exposed.load()) {
            bool clean = false;
            if (int rc = csc_exposed_clean(h, st, false, &clean)) return rc;
            if (!clean) {
                h->last_kernel.store("csc_gather<verify>+csc_repair");
                return csc_repair_apply(h, X, ldx, Y, ldy, batch, st, false, 0);
            }
        }
        bool finite = true, any = false;
        for (size_t q = 0; q < h->host_taps.size(); ++q) finite &= std::isfinite(h->host_taps[q]), any |= tap_stored(h, q);
        const bool band = h->band_tw > 0 && (h->taps_dense || (finite && any && g.k <= 7));
        if (force == kBanded && !band) return fail(SPCONV_EINVAL, "path=banded: geometry unsupported");
        if (!(band && (force == kBanded || (force == kAuto && batch >= 3)))) {
            spb::CscGatherParams cp = csc_params(h, false);
            cp.X = X;
            cp.ldx = ldx;
            cp.Y = Y;
            cp.ldy = ldy;
            cp.batch = (int)batch;
            if (batch <= 2 && cp.inline_taps) {
                // (no PDL right behind the handle's own build: its writes are visible at its end)
                const bool pdl = h->applied.exchange(true);
                CK(spb::launch_csc_gather_lat(cp, st, device_sm_count(), pdl));
                h->last_kernel.store("csc_gather_lat");
                return SPCONV_OK;
            }
            CK(spb::launch_csc_gather(cp, false, st, device_sm_count()));
            h->last_kernel.store("csc_gather");
            return SPCONV_OK;
        }
    }

    // ---- latency path for one or two vectors ----
    const bool spmv_ok = h->k2max <= 49 && !csc;
    if ((force == kSpmv || force == kSpmvPlain) && !spmv_ok)
        return fail(SPCONV_EINVAL, "SPCONV_B200_PATH=spmv: rows longer than 49 entries");
    if (spmv_ok && (force == kSpmv || force == kSpmvPlain || (force == kAuto && batch <= 2))) {
        if (force != kSpmvPlain) {
            spb::SpecParams sp{};
            sp.row_ptr = h->row_ptr;
            sp.col_idx = h->col_idx;
            sp.vals = h->vals;
            sp.ldx = ldx;
            sp.ldy = ldy;
            sp.rows = (int)h->rows;
            sp.nnz = (int)h->nnz;
            sp.m = (int)g.m;
            sp.n = (int)g.n;
            sp.k = (int)g.k;
            sp.s = (int)g.s;
            sp.p = (int)g.p;
            sp.mo = (int)g.mo;
            sp.no = (int)g.no;
            sp.sy = (int)h->sy;
            sp.skew = spb::opt(spb::kOptSpecSkew);
            // closed-form run bounds (conv_run_bounds: k <= 16 lanes); zero taps
            // through the tap mask and W[j] (k <= 7, stored = non-zero double tap)
            bool zt_ok = false;
            if (h->is_conv && !h->taps_dense && g.k <= 7 && !h->host_taps.empty()) {
                bool finite = true, any = false;
                unsigned long long mk = 0;
                for (size_t q = 0; q < h->host_taps.size(); ++q) {
                    finite &= std::isfinite(h->host_taps[q]);
                    const bool stored = h->host_taps64.empty() ? h->host_taps[q] != 0.0f : h->host_taps64[q] != 0.0;
                    if (stored) any = true, mk |= 1ull << q;
                }
                zt_ok = finite && any;
                sp.zt = zt_ok ? 1 : 0;
                sp.nzmask = mk;
                for (int64_t j = 0; zt_ok && j < g.k; ++j) {
                    long long wj = 0;
                    for (int64_t i = 0; i < g.k; ++i) {
                        if (!((mk >> (j * g.k + i)) & 1ull)) continue;
                        const int64_t lo = g.p - i <= 0 ? 0 : (g.p - i + g.s - 1) / g.s;
                        const int64_t hi = g.n + g.p - i - 1 < 0 ? -1 : std::min<int64_t>(g.no - 1, (g.n + g.p - i - 1) / g.s);
                        wj += std::max<int64_t>(0, hi - lo + 1);
                    }
                    sp.zw[j] = wj;
                }
            }
            const bool spec = h->is_conv && (h->taps_dense || zt_ok) && g.k <= 16;
            // Programmatic dependent launch lets the SpMV fetch the matrix before
            // the previous kernel on the stream finishes -- never behind this
            // handle's own build, whose writes are only visible at its end.
            // (nor when the storage was handed out: a kernel of the caller's may
            // have just written it)
            sp.pdl = h->applied.exchange(true) && !h->exposed.load() ? 1 : 0;
            sp.X = X;
            // The windowed kernel (one round trip) wins on matrices that arrive
            // from HBM -- config 2 cold: 12.3 -> 10.2 us; on L2-resident
            // transforms chained back to back the bulk-staged kernel, which
            // prefetches the matrix under the previous kernel (PDL), is faster
            // (config 2 warm 3.0 vs 4.3 us; DenseNet layers 1.0-2.5 vs 1.7-4.7 us;
            // profiles/r02_exp/probe_spmv.txt).  So: the window from 8 MB of
            // matrix up, except in a graph being captured (replays run back to
            // back: the warm case).  Option stage = bulk / window forces either.
            const int stage = spb::opt(spb::kOptStage);
            const bool big = 8.0 * (double)h->nnz >= 8.0 * (1 << 20);
            cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
            if (stage == 0 && big && cudaStreamIsCapturing(st, &cap) != cudaSuccess) {
                cudaGetLastError();  // (legacy stream during another thread's global capture)
                cap = cudaStreamCaptureStatusActive;
            }
            const bool win = spec && spb::spmv_win_ok(sp) &&
                             (stage == 2 || (stage == 0 && big && cap == cudaStreamCaptureStatusNone));
            for (int64_t b0 = 0; b0 < batch; b0 += 2) {  // <= 2 images per launch
                sp.X = X + b0 * ldx;
                sp.Y = Y + b0 * ldy;
                sp.batch = (int)std::min<int64_t>(2, batch - b0);
                CK(win ? spb::launch_spmv_win(sp, h->k2max, st) : spb::launch_spmv_warp(sp, h->k2max, spec, st));
            }
            h->last_kernel.store(win ? "conv_spmv_win" : spec ? "csr_spmv_bulk<spec>" : "csr_spmv_bulk");
            return SPCONV_OK;
        }
        spb::GenericParams gp{h->row_ptr, h->col_idx, h->vals, X, ldx, Y, ldy, (int)h->rows,
                              (int)batch};
        CK(spb::launch_spmv_unrolled(gp, h->k2max, st));
        h->last_kernel.store("csr_spmv_unrolled");
        return SPCONV_OK;
    }

    // ---- band path: CSR band check + register-blocked apply ----
    const bool band_geom = h->is_conv && h->band_tw > 0 && (h->row_ptr || csc);
    if (force == kBanded && !band_geom)
        return fail(SPCONV_EINVAL, "SPCONV_B200_PATH=banded: geometry unsupported");
    const bool band_taps = band_taps_ok(h);
    if (band_geom && (force == kBanded || (force == kAuto && band_taps))) {
        const int sms = device_sm_count();
        spb::BandShape sh{};
        spb::BandParams bp{};
        if (int rc = band_setup(h, csc, false, batch, X, ldx, Y, ldy, bp, sh, sms)) return rc;
        // the apply as a programmatic dependent: its check warps read the
        // matrix before the previous kernel ends -- never right behind the
        // handle's own build, nor over storage handed out to the caller
        bp.pdl = h->applied.exchange(true) && !h->exposed.load() && spb::opt(spb::kOptPdl) != 1 ? 1 : 0;
        CUtensorMap tmap;
        std::memset(&tmap, 0, sizeof tmap);
        RepitchBuf rbuf;
        if (int rc = repitch_for_tma(h, X, ldx, batch, false, bp, sh, &tmap, rbuf, st)) return rc;
        if (!bp.notma && !rbuf.p)
            if (int rc = encode_x_map(&tmap, X, g, ldx, batch, sh.wc, sh.wr, 1, false)) return rc;
        // The fused form -- one kernel: consumers apply with the blocked sums
        // while up to four check warps per CTA verify the storage segment by
        // segment -- where the checks are light: k <= 2, or k = 3 at s = 1
        // (config 3: 256 images 400 -> 362 us, 32 images 77 -> 64 us; pruned
        // k3: 416 -> 388 us).  Heavier checks outweigh the overlap (k5 s1 at 32
        // images: 106 us as two kernels, 126 fused; config 4 at 8 images: 368
        // against 585 us), so there the check runs as a kernel of its own
        // (profiles/r02_exp/ab_forms.txt).  Option "fused" forces either form;
        // the blocked path needs finite taps.
        // Both forms run on the caller's stream only: the check sees exactly
        // the matrix the stream order gives it.
        const int fsel = spb::opt(spb::kOptFused);
        bp.fused = band_taps && bp.seg_div == 1 &&
                           !(csc && spb::band_csc_seg_div((int)g.k, (int)g.s) != 1) &&
                           (fsel ? fsel == 2 : g.k <= 2 || (g.k == 3 && g.s == 1))
                       ? 1
                       : 0;
        if (bp.fused) {
            h->checked.store(true);
            const cudaError_t fe = spb::launch_band((int)g.k, (int)g.s, bp, &tmap, st, nullptr, sms);
            if (fe == cudaSuccess) {
                h->last_kernel.store(csc          ? "conv_spmm_band<fused,csc>"
                                     : bp.fixup ? "conv_spmm_band<fused>+conv_band_fixup"
                                                : "conv_spmm_band<fused>");
                return SPCONV_OK;
            }
            if (fe != cudaErrorNotSupported) CK(fe);
            cudaGetLastError();
            bp.fused = 0;  // this blocking has no fused instantiation
        }
        h->checked.store(true);
        CK(spb::launch_band_check((int)g.k, (int)g.s, bp, st, sms));
        CK(spb::launch_band((int)g.k, (int)g.s, bp, &tmap, st, nullptr, sms));
        h->last_kernel.store(csc ? "conv_band_check<csc>+conv_spmm_band" : "conv_band_check+conv_spmm_band");
        return SPCONV_OK;
    }

    if (csc) return fail(SPCONV_ECUDA, "spconv_spmm: internal error (CSC storage reached the row-major kernels)");

    // ---- tiled (per-entry) path ----
    if (h->is_conv && force != kGeneric) {
        int bt = batch >= 8 ? 8 : batch >= 4 ? 4 : batch >= 2 ? 2 : 1;
        const int k2max = std::max(h->k2max, 1);
        // Tile height: keep the per-CTA (off, val) table <= 64 KB.
        int th = 8;
        while (th > 1 && (size_t)k2max * th * 32 * 8 > 64 * 1024) th >>= 1;
        const int64_t wr = (th - 1) * g.s + g.k;
        const int64_t wc = ((31 * g.s + g.k + 3) + 3) & ~int64_t(3);
        const bool use_tma = tma_ok && wr <= 256 && wc <= 256 && force != kTiledNoTma;
        int stages = use_tma ? 4 : 1;
        size_t smem = 0;
        while (true) {
            smem = spb::tiled_smem_bytes(th, (int)wr, (int)wc, k2max, bt, stages);
            if (smem <= 200 * 1024) break;
            if (stages > 2) --stages;
            else if (bt > 1) bt >>= 1;
            else break;
        }
        if (smem <= 227 * 1024 && g.m < (1ll << 30) && g.n < (1ll << 30)) {
            spb::TiledParams tp{};
            tp.row_ptr = h->row_ptr;
            tp.col_idx = h->col_idx;
            tp.vals = h->vals;
            tp.X = X;
            tp.ldx = ldx;
            tp.Y = Y;
            tp.ldy = ldy;
            tp.batch = (int)batch;
            tp.m = (int)g.m;
            tp.n = (int)g.n;
            tp.s = (int)g.s;
            tp.p = (int)g.p;
            tp.mo = (int)g.mo;
            tp.no = (int)g.no;
            tp.th = th;
            tp.tiles_y = (int)((g.no + 31) / 32);
            tp.wr = (int)wr;
            tp.wc = (int)wc;
            tp.k2max = k2max;
            tp.stages = stages;
            tp.use_tma = use_tma ? 1 : 0;
            CUtensorMap tmap;
            std::memset(&tmap, 0, sizeof tmap);
            if (use_tma)
                if (int rc = encode_x_map(&tmap, X, g, ldx, batch, (int)wc, (int)wr, bt)) return rc;
            CK(spb::launch_tiled(tp, &tmap, bt, smem, st));
            h->last_kernel.store("conv_spmm_tiled");
            return SPCONV_OK;
        }
        if (force == kTiled || force == kTiledNoTma)
            return fail(SPCONV_EINVAL, "SPCONV_B200_PATH=tiled: geometry unsupported");
    }

    // ---- generic CSR path ----
    spb::GenericParams gp{h->row_ptr, h->col_idx, h->vals, X, ldx, Y, ldy, (int)h->rows, (int)batch};
    // the row-block multi-vector kernel (matrix staged once per CTA) for rows
    // of <= 64 entries; SPCONV_B200_GENERIC=plain keeps thread-per-row
    if (h->k2max <= 64 && spb::opt(spb::kOptGeneric) == 0) {
        CK(spb::launch_rowblock(gp, h->k2max, st));
        h->last_kernel.store("csr_spmm_rowblock");
        return SPCONV_OK;
    }
    CK(spb::launch_generic(gp, st));
    h->last_kernel.store("csr_spmm_generic");
    return SPCONV_OK;
}

void free_ws(spconv_csr* h) {
    for (int i = 0; i < 2; ++i) {
        if (h->ws_x[i]) cudaFree(h->ws_x[i]);
        if (h->ws_y[i]) cudaFree(h->ws_y[i]);
        h->ws_x[i] = h->ws_y[i] = nullptr;
    }
    for (int s = 0; s < 3; ++s) {
        for (int i = 0; i < 2; ++i)
            if (h->ws_ev[s][i]) cudaEventDestroy(h->ws_ev[s][i]), h->ws_ev[s][i] = nullptr;
        if (h->ws_stream[s]) cudaStreamDestroy(h->ws_stream[s]), h->ws_stream[s] = nullptr;
    }
    h->ws_chunk = 0;
}

// ---- transform text I/O helpers (inc/conv.hpp:217-244, inc/sparse.hpp:396-432) ----

// Whitespace-separated token reader over a byte range (istream >> semantics
// for well-formed input).
struct TokenReader {
    const char* p;
    const char* e;
    bool ws(char c) const { return c == ' ' || c == '\n' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }
    bool next(std::string_view& tok) {
        while (p < e && ws(*p)) ++p;
        if (p >= e) return false;
        const char* b = p;
        while (p < e && !ws(*p)) ++p;
        tok = std::string_view(b, (size_t)(p - b));
        return true;
    }
    bool i64(int64_t& v) {
        std::string_view t;
        if (!next(t)) return false;
        size_t o = (!t.empty() && t[0] == '+') ? 1 : 0;
        auto r = std::from_chars(t.data() + o, t.data() + t.size(), v);
        return r.ec == std::errc() && r.ptr == t.data() + t.size();
    }
    bool f64(double& v) {  // decimal floating point only (num_get rejects inf / nan / hex)
        std::string_view t;
        if (!next(t)) return false;
        size_t o = (!t.empty() && t[0] == '+') ? 1 : 0;
        for (char c : t.substr(o))
            if (!((c >= '0' && c <= '9') || c == '.' || c == 'e' || c == 'E' || c == '-' || c == '+'))
                return false;
        auto r = std::from_chars(t.data() + o, t.data() + t.size(), v, std::chars_format::general);
        return r.ec == std::errc() && r.ptr == t.data() + t.size();
    }
    std::string_view line() {  // std::getline
        const char* b = p;
        while (p < e && *p != '\n') ++p;
        std::string_view l(b, (size_t)(p - b));
        if (p < e) ++p;
        return l;
    }
    void skip_line() {  // is.ignore(max, '\n')
        while (p < e && *p != '\n') ++p;
        if (p < e) ++p;
    }
};

std::string transform_header(const spconv_csr* h) {
    char buf[256];
    std::snprintf(buf, sizeof buf,
                  "%%%%transform %lld %lld %lld %lld %lld %s\n%%%%sparse coordinate real\n%lld %lld %lld\n",
                  (long long)h->g.m, (long long)h->g.n, (long long)h->g.k, (long long)h->g.s,
                  (long long)h->g.p, h->layout ? "csc" : "csr", (long long)h->rows, (long long)h->cols, (long long)h->nnz);
    return buf;
}

std::string sparse_header(const spconv_csr* h) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "%%%%sparse coordinate real\n%lld %lld %lld\n", (long long)h->rows,
                  (long long)h->cols, (long long)h->nnz);
    return buf;
}

// CSC storage given on the host (already validated), uploaded synchronously.
int attach_csc_host(spconv_csr* h, const std::vector<int32_t>& cp, const std::vector<int32_t>& ci,
                    const std::vector<float>& cv, const double* cv64, cudaStream_t st) {
    const size_t cp_bytes = ((size_t)(h->cols + 1) * 4 + 255) & ~size_t(255);
    const size_t ix_bytes = ((size_t)std::max<int64_t>(h->nnz, 1) * 4 + 255) & ~size_t(255);
    char* mem = nullptr;
    CK(cudaMalloc(&mem, cp_bytes + 2 * ix_bytes + 256));
    h->csc_ptr = reinterpret_cast<int32_t*>(mem);
    h->csc_idx = reinterpret_cast<int32_t*>(mem + cp_bytes);
    h->csc_vals = reinterpret_cast<float*>(mem + cp_bytes + ix_bytes);
    h->layout = 1;
    CK(cudaMemcpyAsync(h->csc_ptr, cp.data(), cp.size() * 4, cudaMemcpyHostToDevice, st));
    if (h->nnz > 0) {
        CK(cudaMemcpyAsync(h->csc_idx, ci.data(), (size_t)h->nnz * 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(h->csc_vals, cv.data(), (size_t)h->nnz * 4, cudaMemcpyHostToDevice, st));
    }
    if (cv64 && h->vals64) {  // exact values (the row-major side found some fp32 cannot hold)
        CK(cudaMalloc(&h->csc_vals64, (size_t)std::max<int64_t>(h->nnz, 1) * 8));
        if (h->nnz > 0)
            CK(cudaMemcpyAsync(h->csc_vals64, cv64, (size_t)h->nnz * 8, cudaMemcpyHostToDevice, st));
    }
    CK(cudaStreamSynchronize(st));  // the host vectors die with the caller
    return SPCONV_OK;
}

// Stable transposition of compressed storage (counting sort on the minor
// index; majors visited ascending), the storage half of relayout
// (inc/sparse.hpp:268-274) for matrices that arrive from the host.
template <class I, class V>
void transpose_host(int64_t major, int64_t minor, const I* ptr, const I* idx, const V* val,
                    std::vector<int32_t>& optr, std::vector<int32_t>& oidx, std::vector<V>& oval) {
    const int64_t nnz = (int64_t)ptr[major];
    optr.assign((size_t)minor + 1, 0);
    oidx.resize((size_t)std::max<int64_t>(nnz, 1));
    oval.resize((size_t)std::max<int64_t>(nnz, 1));
    for (int64_t e = 0; e < nnz; ++e) optr[(size_t)idx[e] + 1]++;
    for (int64_t c = 0; c < minor; ++c) optr[(size_t)c + 1] += optr[(size_t)c];
    std::vector<int32_t> cur(optr.begin(), optr.end() - 1);
    for (int64_t r = 0; r < major; ++r)
        for (int64_t e = (int64_t)ptr[r]; e < (int64_t)ptr[r + 1]; ++e) {
            const int32_t q = cur[(size_t)idx[e]]++;
            oidx[(size_t)q] = (int32_t)r;
            oval[(size_t)q] = val[e];
        }
}


// read_sparse (inc/sparse.hpp:409-432) of the text at R: same header, dims and
// entry checks and messages, compile()'s duplicate rejection in the (major,
// minor) order of the requested layout; returns the row-major arrays.
int parse_sparse(TokenReader& R, bool csc, int64_t& rows, int64_t& cols, std::vector<int64_t>& ptr,
                 std::vector<int64_t>& idx, std::vector<double>& val) {
    std::string header(R.line());
    if (!header.empty() && header.back() == '\r') header.pop_back();
    if (header != "%%sparse coordinate real")
        return fail(SPCONV_ERUNTIME, "read_sparse: bad header line '" + header + "'");
    int64_t nnz;
    if (!R.i64(rows) || !R.i64(cols) || !R.i64(nnz) || rows < 1 || cols < 1 || nnz < 0)
        return fail(SPCONV_ERUNTIME, "read_sparse: bad 'rows cols nnz' line");
    struct Trip {
        int64_t r, c;
        double v;
    };
    std::vector<Trip> t;
    t.reserve((size_t)nnz);
    for (int64_t i = 0; i < nnz; ++i) {
        int64_t r, c;
        double v;
        if (!R.i64(r) || !R.i64(c) || !R.f64(v))
            return fail(SPCONV_ERUNTIME, "read_sparse: expected " + std::to_string(nnz) + " entries, got " +
                                             std::to_string(i));
        if (r - 1 < 0 || r - 1 >= rows || c - 1 < 0 || c - 1 >= cols)
            return fail(SPCONV_EINVAL, "Triplets: entry (" + std::to_string(r - 1) + ", " + std::to_string(c - 1) +
                                           ") outside " + std::to_string(rows) + "x" + std::to_string(cols));
        t.push_back({r - 1, c - 1, v});
    }
    auto by_row = [](const Trip& a, const Trip& b) { return a.r != b.r ? a.r < b.r : a.c < b.c; };
    auto by_col = [](const Trip& a, const Trip& b) { return a.c != b.c ? a.c < b.c : a.r < b.r; };
    if (csc) std::sort(t.begin(), t.end(), by_col);
    else std::sort(t.begin(), t.end(), by_row);
    for (size_t i = 1; i < t.size(); ++i)
        if (t[i].r == t[i - 1].r && t[i].c == t[i - 1].c)
            return fail(SPCONV_EINVAL, "SparseMatrix: duplicate entry at (" + std::to_string(t[i].r) + ", " +
                                           std::to_string(t[i].c) + ")");
    if (csc) std::sort(t.begin(), t.end(), by_row);  // the row-major arrays want (row, col) order
    ptr.assign((size_t)rows + 1, 0);
    idx.resize(t.size());
    val.resize(t.size());
    for (size_t i = 0; i < t.size(); ++i) {
        ptr[(size_t)t[i].r + 1]++;
        idx[i] = t[i].c;
        val[i] = t[i].v;
    }
    for (int64_t r = 0; r < rows; ++r) ptr[(size_t)r + 1] += ptr[(size_t)r];
    return SPCONV_OK;
}
}  // namespace

int spb_fail(int code, const std::string& msg) { return fail(code, msg); }

extern "C" {

const char* spconv_last_error(void) { return g_err.c_str(); }

int spconv_abi_version(void) { return 100; }

int spconv_spec_check(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p) {
    return check_spec(m, n, k, s, p);
}

int spconv_nnz_bound(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int64_t* out) {
    if (int rc = check_spec(m, n, k, s, p)) return rc;
    if (!out) return fail(SPCONV_EINVAL, "spconv_nnz_bound: null output");
    // inc/analysis.hpp:56-66 factorises: (sum_x rows(x)) * (sum_y cols(y)).
    const Geom g = make_geom(m, n, k, s, p);
    int64_t sx = 0, sy = 0, lo, hi;
    for (int64_t x = 0; x < g.mo; ++x) tap_range(x, m, k, s, p, lo, hi), sx += hi - lo;
    for (int64_t y = 0; y < g.no; ++y) tap_range(y, n, k, s, p, lo, hi), sy += hi - lo;
    *out = sx * sy;
    return SPCONV_OK;
}

// Exact-fp64 fill of a tag build (spconv_build_transform_f64): device tables
// of the taps' fp32 / fp64 values; `done` = the build kernel wrote vals64.
struct F64Fill {
    const float* t32;   // host k*k
    const double* t64;  // host k*k
    bool done;
};

static int build_csr_impl(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, const float* kernel_kxk, int device,
                          void* stream, spconv_csr** out, F64Fill* f64);

int spconv_build_csr(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p,
                     const float* kernel_kxk, int device, void* stream, spconv_csr** out) {
    return build_csr_impl(m, n, k, s, p, kernel_kxk, device, stream, out, nullptr);
}

static int build_csr_impl(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, const float* kernel_kxk, int device,
                          void* stream, spconv_csr** out, F64Fill* f64) {
    if (int rc = check_spec(m, n, k, s, p)) return rc;
    if (!kernel_kxk || !out) return fail(SPCONV_EINVAL, "spconv_build_csr: null argument");
    *out = nullptr;
    const Geom g = make_geom(m, n, k, s, p);
    if (m * n >= (1ll << 31) || g.mo * g.no >= (1ll << 31))
        return fail(SPCONV_EINVAL, "spconv_build_csr: " + spec_str(m, n, k, s, p) +
                                       " exceeds the int32 device index range");
    HostTables ht;
    make_tables(g, kernel_kxk, ht);
    if (ht.nnz >= (1ll << 31))
        return fail(SPCONV_EINVAL, "spconv_build_csr: nnz " + std::to_string(ht.nnz) +
                                       " exceeds the int32 device index range");
    DeviceGuard dg(device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    keep_pool_memory(device);

    auto* h = new (std::nothrow) spconv_csr();
    if (!h) return fail(SPCONV_ECUDA, "out of host memory");
    h->device = device;
    h->is_conv = true;
    h->g = g;
    h->rows = g.mo * g.no;
    h->cols = m * n;
    h->nnz = ht.nnz;
    h->k2max = (int)ht.k2max;

    h->taps_dense = ht.dense;
    h->host_taps.assign(kernel_kxk, kernel_kxk + k * k);
    {
        int64_t lo, hi;
        for (int64_t yy = 0; yy < g.no; ++yy) tap_range(yy, g.n, g.k, g.s, g.p, lo, hi), h->sy += hi - lo;
    }
    h->fail_flag = flag_alloc();  // (the fused band apply's verdict word)
    if (!h->fail_flag) {
        delete h;
        return fail(SPCONV_ECUDA, "cudaHostAlloc(verdict words) failed");
    }

    // One stream-ordered allocation for the CSR (+256 B slack so prologue
    // reads one-past-the-end stay in bounds).
    const size_t rp_bytes = ((size_t)(h->rows + 1) * 4 + 255) & ~size_t(255);
    const size_t ix_bytes = ((size_t)std::max<int64_t>(ht.nnz, 1) * 4 + 255) & ~size_t(255);
    const size_t tap_bytes = ((size_t)(k * k) * 4 + 255) & ~size_t(255);
    size_t seg_bytes = 0;
    if (spb::band_supported((int)k, (int)s)) {
        h->band_tw = spb::band_tile_width((int)k, (int)s);
        const int64_t segw = h->band_tw / spb::band_seg_div((int)k, (int)s);
        seg_bytes = ((size_t)(g.mo * ((g.no + segw - 1) / segw)) + 255) & ~size_t(255);
    }
    char* csr = nullptr;
    cudaError_t e = cudaMallocAsync(&csr, rp_bytes + 2 * ix_bytes + 256 + tap_bytes + seg_bytes, st);
    if (e != cudaSuccess) {
        flag_free(h->fail_flag);
        delete h;
        return cuda_fail(e, "cudaMallocAsync(CSR)");
    }
    h->row_ptr = reinterpret_cast<int32_t*>(csr);
    h->col_idx = reinterpret_cast<int32_t*>(csr + rp_bytes);
    h->vals = reinterpret_cast<float*>(csr + rp_bytes + ix_bytes);
    h->taps = reinterpret_cast<float*>(csr + rp_bytes + 2 * ix_bytes + 256);
    if (seg_bytes) h->seg_ok = reinterpret_cast<uint8_t*>(csr + rp_bytes + 2 * ix_bytes + 256 + tap_bytes);

    spb::BuildParams bp{};
    bp.m = (int)m;
    bp.n = (int)n;
    bp.k = (int)k;
    bp.s = (int)s;
    bp.p = (int)p;
    bp.mo = (int)g.mo;
    bp.no = (int)g.no;
    bp.rows = (int)h->rows;
    bp.row_ptr = h->row_ptr;
    bp.col_idx = h->col_idx;
    bp.vals = h->vals;
    bp.taps_out = h->taps;
    bp.nnz_total = ht.nnz;
    bp.bulk_store = spb::opt(spb::kOptBulkStoreOff) ? 0 : 1;
    char* tab = nullptr;
    if (k <= spb::kSmallK) {  // tables ride in the kernel parameters: no copies, no allocation
        bp.small = 1;
        std::copy(ht.taps.begin(), ht.taps.end(), bp.tab.taps);
        std::copy(ht.sat.begin(), ht.sat.end(), bp.tab.sat);
        std::copy(ht.w.begin(), ht.w.end(), bp.tab.w);
    } else {
        const size_t taps_b = ((ht.taps.size() * 4) + 255) & ~size_t(255);
        const size_t sat_b = ((ht.sat.size() * 4) + 255) & ~size_t(255);
        const size_t w_b = ht.w.size() * 8;
        e = cudaMallocAsync(&tab, taps_b + sat_b + w_b, st);
        if (e != cudaSuccess) {
            cudaFreeAsync(csr, st);
            flag_free(h->fail_flag);
            delete h;
            return cuda_fail(e, "cudaMallocAsync(tables)");
        }
        // Pageable copies are staged by the driver before the call returns.
        cudaMemcpyAsync(tab, ht.taps.data(), ht.taps.size() * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(tab + taps_b, ht.sat.data(), ht.sat.size() * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(tab + taps_b + sat_b, ht.w.data(), w_b, cudaMemcpyHostToDevice, st);
        bp.small = 0;
        bp.t.taps = reinterpret_cast<const float*>(tab);
        bp.t.sat = reinterpret_cast<const int32_t*>(tab + taps_b);
        bp.t.w = reinterpret_cast<const long long*>(tab + taps_b + sat_b);
    }
    // Stage entries through shared memory when a CTA's worst case fits.
    const int64_t k2 = k * k;
    int block = 256;
    while (block > 64 && (size_t)block * k2 * 8 > 64 * 1024) block >>= 1;
    const size_t tab_bytes = (size_t)(((k + 1) * (k + 1) + k2 + 3) & ~int64_t(3)) * 4;
    size_t smem = tab_bytes;
    bp.stage = 0;
    if ((size_t)block * k2 * 8 <= 96 * 1024 && tab_bytes <= 64 * 1024) {
        bp.stage = 1;
        bp.stage_words = (int)((block * k2 + 3 + 3) & ~int64_t(3));
        smem += (size_t)bp.stage_words * 4 * 2;
    } else {
        block = 256;
    }
    if (smem > 200 * 1024) {
        if (tab) cudaFreeAsync(tab, st);
        cudaFreeAsync(csr, st);
        flag_free(h->fail_flag);
        delete h;
        return fail(SPCONV_EINVAL, "spconv_build_csr: kernel side " + std::to_string(k) +
                                       " too large for the device build");
    }
    if (f64) {  // exact values: vals64 (written by the fill, or by the caller's retag pass)
        e = cudaMallocAsync(&h->vals64, (size_t)std::max<int64_t>(ht.nnz, 1) * 8, st);
        if (k * k <= 121) {  // the fill's tables ride in the parameters (k <= 11)
            std::copy(f64->t32, f64->t32 + k * k, bp.f64_t32);
            std::copy(f64->t64, f64->t64 + k * k, bp.f64_t64);
            bp.vals64 = h->vals64;
        }
    }
    bool f64_done = false;
    if (e == cudaSuccess) e = spb::launch_csr_build(bp, ht.nonzero, block, smem, &f64_done, st);
    if (f64) f64->done = f64_done;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (e == cudaSuccess) e = cudaStreamIsCapturing(st, &cap);
    if (e == cudaSuccess && cap == cudaStreamCaptureStatusNone) {  // (a captured build has no event)
        e = cudaEventCreateWithFlags(&h->built, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(h->built, st);
    }
    if (tab) cudaFreeAsync(tab, st);
    if (e != cudaSuccess) {
        if (h->built) cudaEventDestroy(h->built);
        if (h->vals64) cudaFreeAsync(h->vals64, st);
        cudaFreeAsync(csr, st);
        cudaStreamSynchronize(st);
        flag_free(h->fail_flag);
        delete h;
        return cuda_fail(e, "csr_build launch");
    }
    *out = h;
    return SPCONV_OK;
}

static int relayout_host(const spconv_csr* h, int layout, void* stream, spconv_csr** out);

// Kernel sides beyond the CSC kernels' 32 (k > 32): the CSR built on the device,
// its CSC storage by the host transposition (a generic CSC handle, applied
// through its row-major arrays).  Replaces *io.
static int csc_of_wide_kernel(spconv_csr** io, void* stream) {
    spconv_csr* c = nullptr;
    const int rc = relayout_host(*io, 1, stream, &c);
    spconv_csr_free(*io);
    *io = c;
    return rc;
}

// build_transform(kernel, spec, Layout::CSC): the CSC storage only, built in
// closed form on the device (csc_build.cu); no row-major arrays -- the apply
// kernels read the CSC storage (csc_apply.cu, conv_band_check<csc>).
static int build_csc_impl(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, const float* kernel_kxk, int device,
                          void* stream, spconv_csr** out) {
    if (int rc = check_spec(m, n, k, s, p)) return rc;
    if (!kernel_kxk || !out) return fail(SPCONV_EINVAL, "spconv_build_transform: null argument");
    *out = nullptr;
    const Geom g = make_geom(m, n, k, s, p);
    if (m * n >= (1ll << 31) || g.mo * g.no >= (1ll << 31))
        return fail(SPCONV_EINVAL, "spconv_build_transform: " + spec_str(m, n, k, s, p) +
                                       " exceeds the int32 device index range");
    HostTables ht;
    make_tables(g, kernel_kxk, ht);
    if (ht.nnz >= (1ll << 31))
        return fail(SPCONV_EINVAL, "spconv_build_transform: nnz " + std::to_string(ht.nnz) +
                                       " exceeds the int32 device index range");
    DeviceGuard dg(device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    keep_pool_memory(device);
    auto* h = new (std::nothrow) spconv_csr();
    if (!h) return fail(SPCONV_ECUDA, "out of host memory");
    h->device = device;
    h->is_conv = true;
    h->layout = 1;
    h->g = g;
    h->rows = g.mo * g.no;
    h->cols = m * n;
    h->nnz = ht.nnz;
    h->k2max = (int)ht.k2max;
    h->taps_dense = ht.dense;
    h->host_taps.assign(kernel_kxk, kernel_kxk + k * k);
    {
        int64_t lo, hi;
        for (int64_t yy = 0; yy < g.no; ++yy) tap_range(yy, g.n, g.k, g.s, g.p, lo, hi), h->sy += hi - lo;
    }
    h->fail_flag = flag_alloc();
    if (!h->fail_flag) {
        delete h;
        return fail(SPCONV_ECUDA, "cudaHostAlloc(verdict words) failed");
    }
    const size_t cp_bytes = ((size_t)(h->cols + 1) * 4 + 255) & ~size_t(255);
    const size_t ix_bytes = ((size_t)std::max<int64_t>(ht.nnz, 1) * 4 + 255) & ~size_t(255);
    const size_t tap_bytes = ((size_t)(k * k) * 4 + 255) & ~size_t(255);
    size_t seg_bytes = 0;
    if (spb::band_supported((int)k, (int)s)) {  // CSC segments: one input row x s * band_tw input columns
        h->band_tw = spb::band_tile_width((int)k, (int)s);
        const int64_t segw = h->band_tw / spb::band_csc_seg_div((int)k, (int)s);
        h->csc_tiles_b = (int)((n + segw * s - 1) / (segw * s));  // (segments of s * segment-width columns)
        seg_bytes = ((size_t)(m * h->csc_tiles_b) + 255) & ~size_t(255);
    }
    char* mem = nullptr;
    cudaError_t e = cudaMallocAsync(&mem, cp_bytes + 2 * ix_bytes + 256 + tap_bytes + seg_bytes, st);
    if (e != cudaSuccess) {
        flag_free(h->fail_flag);
        delete h;
        return cuda_fail(e, "cudaMallocAsync(CSC)");
    }
    h->csc_ptr = reinterpret_cast<int32_t*>(mem);
    h->csc_idx = reinterpret_cast<int32_t*>(mem + cp_bytes);
    h->csc_vals = reinterpret_cast<float*>(mem + cp_bytes + ix_bytes);
    h->taps = reinterpret_cast<float*>(mem + cp_bytes + 2 * ix_bytes + 256);
    if (seg_bytes) h->seg_ok = reinterpret_cast<uint8_t*>(mem + cp_bytes + 2 * ix_bytes + 256 + tap_bytes);
    // (pageable source: staged by the driver before the call returns)
    e = cudaMemcpyAsync(h->taps, kernel_kxk, (size_t)(k * k) * 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        spb::CscParams cp{};
        cp.m = (int)g.m;
        cp.n = (int)g.n;
        cp.k = (int)g.k;
        cp.s = (int)g.s;
        cp.p = (int)g.p;
        cp.mo = (int)g.mo;
        cp.no = (int)g.no;
        cp.cols = (int)h->cols;
        cp.taps = h->taps;
        cp.col_ptr = h->csc_ptr;
        cp.row_idx = h->csc_idx;
        cp.vals = h->csc_vals;
        cp.bulk_store = spb::opt(spb::kOptBulkStoreOff) ? 0 : 1;
        const int64_t per_axis = std::min<int64_t>(g.k, (g.k + g.s - 1) / g.s);
        e = spb::launch_csc_build(cp, (int)(per_axis * per_axis), ht.nonzero, st);
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (e == cudaSuccess) e = cudaStreamIsCapturing(st, &cap);
    if (e == cudaSuccess && cap == cudaStreamCaptureStatusNone) {
        e = cudaEventCreateWithFlags(&h->built, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(h->built, st);
    }
    if (e != cudaSuccess) {
        if (h->built) cudaEventDestroy(h->built);
        cudaFreeAsync(mem, st);
        cudaStreamSynchronize(st);
        flag_free(h->fail_flag);
        delete h;
        return cuda_fail(e, "csc_build launch");
    }
    *out = h;
    return SPCONV_OK;
}

int spconv_build_transform(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p,
                           const float* kernel_kxk, int layout, int device, void* stream,
                           spconv_csr** out) {
    if (layout != 0 && layout != 1)
        return fail(SPCONV_EINVAL, "spconv_build_transform: layout must be 0 (csr) or 1 (csc)");
    if (layout == 1 && k <= 32) return build_csc_impl(m, n, k, s, p, kernel_kxk, device, stream, out);
    if (int rc = spconv_build_csr(m, n, k, s, p, kernel_kxk, device, stream, out)) return rc;
    if (layout == 0) return SPCONV_OK;
    return csc_of_wide_kernel(out, stream);
}

int spconv_build_transform_f64(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p,
                               const double* kernel_kxk, int layout, int device, void* stream,
                               spconv_csr** out) {
    if (layout != 0 && layout != 1)
        return fail(SPCONV_EINVAL, "spconv_build_transform_f64: layout must be 0 (csr) or 1 (csc)");
    if (int rc = check_spec(m, n, k, s, p)) return rc;
    if (!kernel_kxk || !out) return fail(SPCONV_EINVAL, "spconv_build_transform_f64: null argument");
    *out = nullptr;
    const int64_t kk = k * k;
    if (kk >= (1ll << 24))
        return fail(SPCONV_EINVAL, "spconv_build_transform_f64: kernel side " + std::to_string(k) + " too large");
    std::vector<float> t32((size_t)kk);
    bool exact = true;
    for (int64_t q = 0; q < kk; ++q) {
        t32[(size_t)q] = (float)kernel_kxk[q];
        exact &= __builtin_bit_cast(uint64_t, (double)t32[(size_t)q]) == __builtin_bit_cast(uint64_t, kernel_kxk[q]);
    }
    if (exact)  // every tap is an fp32 number: the fp32 build is already exact
        return spconv_build_transform(m, n, k, s, p, t32.data(), layout, device, stream, out);
    // Build the structure from tags (q + 1 where the DOUBLE tap is non-zero,
    // inc/sparse.hpp:335).  The persistent build (k <= 5) writes the real fp32
    // values and the exact doubles from its staging; other builds get a
    // tag -> value pass afterwards (retag_kernel).
    std::vector<float> tag((size_t)kk);
    for (int64_t q = 0; q < kk; ++q) tag[(size_t)q] = kernel_kxk[q] != 0.0 ? (float)(q + 1) : 0.0f;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    F64Fill fill{t32.data(), kernel_kxk, false};
    spconv_csr* h = nullptr;
    // (argument and int32-range checks first, inside: no device work before them)
    if (layout == 1 && k > 32) {  // (see csc_of_wide_kernel)
        if (int rc = spconv_build_transform_f64(m, n, k, s, p, kernel_kxk, 0, device, stream, &h)) return rc;
        if (int rc = csc_of_wide_kernel(&h, stream)) return rc;
        *out = h;
        return SPCONV_OK;
    }
    if (layout == 1) {  // CSC storage only, from the tags
        if (int rc = build_csc_impl(m, n, k, s, p, tag.data(), device, stream, &h)) return rc;
    } else {
        if (int rc = build_csr_impl(m, n, k, s, p, tag.data(), device, stream, &h, &fill)) return rc;
    }
    DeviceGuard dg(device);
    int rc = SPCONV_OK;
    // device tables of the values for the retag passes (none needed when the
    // fill wrote them and there is no CSC storage)
    const bool need_tables = !fill.done || h->layout == 1;
    const size_t t32_bytes = ((size_t)kk * 4 + 255) & ~size_t(255);
    char* tt = nullptr;
    cudaError_t e = rc || !need_tables ? cudaSuccess : cudaMallocAsync(&tt, t32_bytes + (size_t)kk * 8, st);
    const float* d32 = reinterpret_cast<const float*>(tt);
    const double* d64 = reinterpret_cast<const double*>(tt + t32_bytes);
    // (pageable sources: staged by the driver before each call returns)
    if (!rc && e == cudaSuccess && need_tables) e = cudaMemcpyAsync(tt, t32.data(), (size_t)kk * 4, cudaMemcpyHostToDevice, st);
    if (!rc && e == cudaSuccess && need_tables)
        e = cudaMemcpyAsync(tt + t32_bytes, kernel_kxk, (size_t)kk * 8, cudaMemcpyHostToDevice, st);
    const size_t vb = (size_t)std::max<int64_t>(h->nnz, 1) * 8;
    if (rc == SPCONV_OK && e == cudaSuccess && h->layout == 0 && !fill.done)
        e = spb::launch_retag(h->vals, h->vals64, h->nnz, d32, d64, st);
    if (rc == SPCONV_OK && e == cudaSuccess && h->layout == 1) {
        e = cudaMallocAsync(&h->csc_vals64, vb, st);
        if (e == cudaSuccess) e = spb::launch_retag(h->csc_vals, h->csc_vals64, h->nnz, d32, d64, st);
    }
    // the exact taps on the device (the fp64 band sums, the CSC kernels' fp64 checks and sums)
    if (rc == SPCONV_OK && e == cudaSuccess) e = cudaMallocAsync(&h->taps64, (size_t)kk * 8, st);
    if (rc == SPCONV_OK && e == cudaSuccess)  // (pageable source: staged before the call returns)
        e = cudaMemcpyAsync(h->taps64, kernel_kxk, (size_t)kk * 8, cudaMemcpyHostToDevice, st);
    // the device taps (band check, CSC rebuilds) become the real fp32 taps
    if (rc == SPCONV_OK && e == cudaSuccess)
        e = need_tables ? cudaMemcpyAsync(h->taps, d32, (size_t)kk * 4, cudaMemcpyDeviceToDevice, st)
                        : cudaMemcpyAsync(h->taps, t32.data(), (size_t)kk * 4, cudaMemcpyHostToDevice, st);
    if (rc == SPCONV_OK && e == cudaSuccess && h->built) e = cudaEventRecord(h->built, st);  // host-buffer calls see the values
    if (tt) cudaFreeAsync(tt, st);
    if (rc != SPCONV_OK || e != cudaSuccess) {
        const std::string msg = rc ? g_err : std::string();
        spconv_csr_free(h);
        return rc ? fail(rc, msg) : cuda_fail(e, "spconv_build_transform_f64");
    }
    h->host_taps = t32;
    h->host_taps64.assign(kernel_kxk, kernel_kxk + kk);
    h->taps_dense = true;
    for (float v : t32) h->taps_dense &= v != 0.0f && std::isfinite(v);
    *out = h;
    return SPCONV_OK;
}

int spconv_csr_layout(const spconv_csr* h, int* layout) {
    if (!h || !layout) return fail(SPCONV_EINVAL, "null argument");
    *layout = h->layout;
    return SPCONV_OK;
}

int spconv_matrix_from_host(int64_t rows, int64_t cols, int layout, const int64_t* ptr,
                            const int64_t* idx, const double* vals, int device, void* stream,
                            spconv_csr** out) {
    if (layout == 0) return spconv_csr_from_host(rows, cols, ptr, idx, vals, device, stream, out);
    if (layout != 1) return fail(SPCONV_EINVAL, "spconv_matrix_from_host: layout must be 0 (csr) or 1 (csc)");
    if (!out || !ptr) return fail(SPCONV_EINVAL, "spconv_matrix_from_host: null argument");
    *out = nullptr;
    if (rows < 1 || cols < 1)
        return fail(SPCONV_EINVAL, "Triplets: dimensions must be at least 1x1, got " +
                                       std::to_string(rows) + "x" + std::to_string(cols));
    if (rows >= (1ll << 31) || cols >= (1ll << 31))
        return fail(SPCONV_EINVAL, "spconv_matrix_from_host: dimensions exceed the int32 range");
    const int64_t nnz = ptr[cols];
    if (ptr[0] != 0 || nnz < 0 || nnz >= (1ll << 31))
        return fail(SPCONV_EINVAL, "spconv_matrix_from_host: bad col_ptr");
    for (int64_t c = 0; c < cols; ++c) {
        if (ptr[c + 1] < ptr[c]) return fail(SPCONV_EINVAL, "spconv_matrix_from_host: col_ptr not non-decreasing");
        for (int64_t e = ptr[c]; e < ptr[c + 1]; ++e)
            if (idx[e] < 0 || idx[e] >= rows || (e > ptr[c] && idx[e] <= idx[e - 1]))
                return fail(SPCONV_EINVAL, "spconv_matrix_from_host: row indices must be in range "
                                           "and strictly ascending per column");
    }
    // row-major arrays for the kernels: the transposed storage
    std::vector<int32_t> rp, ri;
    std::vector<double> rv;
    transpose_host(cols, rows, ptr, idx, vals, rp, ri, rv);
    std::vector<int64_t> rp64(rp.begin(), rp.end()), ri64(ri.begin(), ri.end());
    spconv_csr* h = nullptr;
    if (int rc = spconv_csr_from_host(rows, cols, rp64.data(), ri64.data(), rv.data(), device, stream, &h))
        return rc;
    std::vector<int32_t> cp((size_t)cols + 1), ci((size_t)std::max<int64_t>(nnz, 1));
    std::vector<float> cv((size_t)std::max<int64_t>(nnz, 1));
    for (int64_t c = 0; c <= cols; ++c) cp[(size_t)c] = (int32_t)ptr[c];
    for (int64_t e = 0; e < nnz; ++e) ci[(size_t)e] = (int32_t)idx[e], cv[(size_t)e] = (float)vals[e];
    DeviceGuard dg(device);
    if (int rc = attach_csc_host(h, cp, ci, cv, vals, static_cast<cudaStream_t>(stream))) {
        const std::string msg = g_err;
        spconv_csr_free(h);
        return fail(rc, msg);
    }
    *out = h;
    return SPCONV_OK;
}

// spconv_csr_export of the row-major arrays whatever h's layout (a non-owning view).
static int export_row_major(const spconv_csr* h, int64_t* rp, int64_t* ri, double* rv) {
    spconv_csr tmp;
    tmp.device = h->device;
    tmp.rows = h->rows;
    tmp.cols = h->cols;
    tmp.nnz = h->nnz;
    tmp.row_ptr = h->row_ptr;
    tmp.col_idx = h->col_idx;
    tmp.vals = h->vals;
    tmp.vals64 = h->vals64;
    return spconv_csr_export(&tmp, rp, ri, rv);
}

static int relayout_host(const spconv_csr* h, int layout, void* stream, spconv_csr** out);

int spconv_relayout(const spconv_csr* h, int layout, void* stream, spconv_csr** out) {
    if (!h || !out) return fail(SPCONV_EINVAL, "spconv_relayout: null argument");
    if (layout != 0 && layout != 1) return fail(SPCONV_EINVAL, "spconv_relayout: layout must be 0 (csr) or 1 (csc)");
    *out = nullptr;
    if (h->is_conv && !h->host_taps.empty()) {
        // A conv handle IS the transform of its taps: rebuild in the target
        // layout on the device (closed form; no host round trip).
        const Geom& g = h->g;
        if (!h->host_taps64.empty())
            return spconv_build_transform_f64(g.m, g.n, g.k, g.s, g.p, h->host_taps64.data(), layout, h->device,
                                              stream, out);
        return spconv_build_transform(g.m, g.n, g.k, g.s, g.p, h->host_taps.data(), layout, h->device,
                                      stream, out);
    }
    return relayout_host(h, layout, stream, out);
}

// Matrices that came from the host: transposition of the host copy.
static int relayout_host(const spconv_csr* h, int layout, void* stream, spconv_csr** out) {
    std::vector<int64_t> rp((size_t)h->rows + 1), ri((size_t)std::max<int64_t>(h->nnz, 1));
    std::vector<double> rv((size_t)std::max<int64_t>(h->nnz, 1));
    if (int rc = export_row_major(h, rp.data(), ri.data(), rv.data())) return rc;
    int rc;
    if (layout == 0) {
        rc = spconv_csr_from_host(h->rows, h->cols, rp.data(), ri.data(), rv.data(), h->device, stream, out);
    } else {
        std::vector<int32_t> cp, ci;
        std::vector<double> cv;
        transpose_host(h->rows, h->cols, rp.data(), ri.data(), rv.data(), cp, ci, cv);
        std::vector<int64_t> cp64(cp.begin(), cp.end()), ci64(ci.begin(), ci.end());
        rc = spconv_matrix_from_host(h->rows, h->cols, 1, cp64.data(), ci64.data(), cv.data(), h->device,
                                     stream, out);
    }
    if (rc == SPCONV_OK) (*out)->g = h->g;  // geometry travels with the matrix
    return rc;
}

int spconv_csr_from_host(int64_t rows, int64_t cols, const int64_t* row_ptr,
                         const int64_t* col_idx, const double* vals, int device, void* stream,
                         spconv_csr** out) {
    if (!out || !row_ptr) return fail(SPCONV_EINVAL, "spconv_csr_from_host: null argument");
    *out = nullptr;
    if (rows < 1 || cols < 1)
        return fail(SPCONV_EINVAL, "Triplets: dimensions must be at least 1x1, got " +
                                       std::to_string(rows) + "x" + std::to_string(cols));
    if (rows >= (1ll << 31) || cols >= (1ll << 31))
        return fail(SPCONV_EINVAL, "spconv_csr_from_host: dimensions exceed the int32 range");
    const int64_t nnz = row_ptr[rows];
    if (row_ptr[0] != 0 || nnz < 0 || nnz >= (1ll << 31))
        return fail(SPCONV_EINVAL, "spconv_csr_from_host: bad row_ptr");
    std::vector<int32_t> rp((size_t)rows + 1), ci((size_t)std::max<int64_t>(nnz, 1));
    std::vector<float> vv((size_t)std::max<int64_t>(nnz, 1));
    int64_t k2max = 0;
    for (int64_t r = 0; r < rows; ++r) {
        if (row_ptr[r + 1] < row_ptr[r])
            return fail(SPCONV_EINVAL, "spconv_csr_from_host: row_ptr not non-decreasing");
        k2max = std::max(k2max, row_ptr[r + 1] - row_ptr[r]);
        for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
            if (col_idx[e] < 0 || col_idx[e] >= cols || (e > row_ptr[r] && col_idx[e] <= col_idx[e - 1]))
                return fail(SPCONV_EINVAL, "spconv_csr_from_host: column indices must be in range "
                                           "and strictly ascending per row");
        }
        rp[r] = (int32_t)row_ptr[r];
    }
    rp[rows] = (int32_t)nnz;
    bool exact = true;
    for (int64_t e = 0; e < nnz; ++e) {
        ci[e] = (int32_t)col_idx[e], vv[e] = (float)vals[e];
        exact &= __builtin_bit_cast(uint64_t, (double)vv[e]) == __builtin_bit_cast(uint64_t, vals[e]);
    }
    DeviceGuard dg(device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    auto* h = new (std::nothrow) spconv_csr();
    if (!h) return fail(SPCONV_ECUDA, "out of host memory");
    h->device = device;
    h->rows = rows;
    h->cols = cols;
    h->nnz = nnz;
    h->k2max = (int)k2max;
    const size_t rp_bytes = ((size_t)(rows + 1) * 4 + 255) & ~size_t(255);
    const size_t ix_bytes = (ci.size() * 4 + 255) & ~size_t(255);
    char* csr = nullptr;
    // +256 B: 16-byte bulk copies round a run's end up by up to 12 bytes
    cudaError_t e = cudaMalloc(&csr, rp_bytes + 2 * ix_bytes + 256);
    if (e != cudaSuccess) {
        delete h;
        return cuda_fail(e, "cudaMalloc(CSR)");
    }
    h->row_ptr = reinterpret_cast<int32_t*>(csr);
    h->col_idx = reinterpret_cast<int32_t*>(csr + rp_bytes);
    h->vals = reinterpret_cast<float*>(csr + rp_bytes + ix_bytes);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    e = cudaMemcpyAsync(h->row_ptr, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(h->col_idx, ci.data(), ci.size() * 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(h->vals, vv.data(), vv.size() * 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && !exact) {  // keep the exact values next to the fp32 ones
        e = cudaMalloc(&h->vals64, (size_t)std::max<int64_t>(nnz, 1) * 8);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h->vals64, vals, (size_t)nnz * 8, cudaMemcpyHostToDevice, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // host vectors die here
    if (e != cudaSuccess) {
        cudaFree(csr);
        if (h->vals64) cudaFree(h->vals64);
        delete h;
        return cuda_fail(e, "spconv_csr_from_host upload");
    }
    *out = h;
    return SPCONV_OK;
}

int spconv_matrix_from_coo(int64_t rows, int64_t cols, int64_t n, const int64_t* row, const int64_t* col,
                           const double* vals, int layout, int device, void* stream, spconv_csr** out) {
    if (!out) return fail(SPCONV_EINVAL, "spconv_matrix_from_coo: null argument");
    *out = nullptr;
    if (layout != 0 && layout != 1) return fail(SPCONV_EINVAL, "spconv_matrix_from_coo: layout must be 0 (csr) or 1 (csc)");
    if (rows < 1 || cols < 1)
        return fail(SPCONV_EINVAL, "Triplets: dimensions must be at least 1x1, got " + std::to_string(rows) + "x" +
                                       std::to_string(cols));
    if (rows >= (1ll << 31) || cols >= (1ll << 31) || n < 0 || n >= (1ll << 31))
        return fail(SPCONV_EINVAL, "spconv_matrix_from_coo: sizes exceed the int32 range");
    if (n > 0 && (!row || !col || !vals)) return fail(SPCONV_EINVAL, "spconv_matrix_from_coo: null argument");
    bool exact = true;
    for (int64_t i = 0; i < n; ++i) {  // Triplets::add's range check (inc/sparse.hpp:55-62)
        if (row[i] < 0 || row[i] >= rows || col[i] < 0 || col[i] >= cols)
            return fail(SPCONV_EINVAL, "Triplets: entry (" + std::to_string(row[i]) + ", " + std::to_string(col[i]) +
                                           ") outside " + std::to_string(rows) + "x" + std::to_string(cols));
        exact &= __builtin_bit_cast(uint64_t, (double)(float)vals[i]) == __builtin_bit_cast(uint64_t, vals[i]);
    }
    DeviceGuard dg(device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto* h = new (std::nothrow) spconv_csr();
    if (!h) return fail(SPCONV_ECUDA, "out of host memory");
    h->device = device;
    h->rows = rows;
    h->cols = cols;
    h->nnz = n;
    // (major+1 ptr, idx, vals: same slack conventions as spconv_csr_from_host)
    auto alloc = [&](int64_t major, int32_t** p, int32_t** ix, float** v, double** v64) -> cudaError_t {
        const size_t pb = ((size_t)(major + 1) * 4 + 255) & ~size_t(255);
        const size_t ib = ((size_t)std::max<int64_t>(n, 1) * 4 + 255) & ~size_t(255);
        char* mem = nullptr;
        cudaError_t e = cudaMalloc(&mem, pb + 2 * ib + 256);
        if (e != cudaSuccess) return e;
        *p = reinterpret_cast<int32_t*>(mem);
        *ix = reinterpret_cast<int32_t*>(mem + pb);
        *v = reinterpret_cast<float*>(mem + pb + ib);
        if (!exact) e = cudaMalloc(v64, (size_t)std::max<int64_t>(n, 1) * 8);
        return e;
    };
    long long dup = -1;
    int64_t dr = 0, dc = 0;
    int maxlen = 0, unused = 0;
    cudaError_t e = cudaSuccess;
    if (layout == 1) {  // the storage order first: compile() reports the first duplicate in it
        h->layout = 1;
        e = alloc(cols, &h->csc_ptr, &h->csc_idx, &h->csc_vals, &h->csc_vals64);
        if (e == cudaSuccess)
            e = spb::coo_compile(n, row, col, vals, rows, cols, false, h->csc_ptr, h->csc_idx, h->csc_vals,
                                 h->csc_vals64, &dup, &dr, &dc, &unused, st);
    }
    // the row-major arrays every apply kernel reads
    if (e == cudaSuccess && dup < 0) e = alloc(rows, &h->row_ptr, &h->col_idx, &h->vals, &h->vals64);
    if (e == cudaSuccess && dup < 0)
        e = spb::coo_compile(n, row, col, vals, rows, cols, true, h->row_ptr, h->col_idx, h->vals, h->vals64, &dup,
                             &dr, &dc, &maxlen, st);
    h->k2max = maxlen;
    if (e != cudaSuccess || dup >= 0) {
        spconv_csr_free(h);
        if (e != cudaSuccess) return cuda_fail(e, "spconv_matrix_from_coo");
        return fail(SPCONV_EINVAL, "SparseMatrix: duplicate entry at (" + std::to_string(dr) + ", " + std::to_string(dc) + ")");
    }
    *out = h;
    return SPCONV_OK;
}

// A generic handle with row-major arrays for `nnz` entries over rows x cols
// (+ fp64 values when `exact64`), same slack conventions as the uploads.
static int new_generic(int64_t rows, int64_t cols, int64_t nnz, bool exact64, int device, spconv_csr** out) {
    auto* h = new (std::nothrow) spconv_csr();
    if (!h) return fail(SPCONV_ECUDA, "out of host memory");
    h->device = device;
    h->rows = rows;
    h->cols = cols;
    h->nnz = nnz;
    const size_t pb = ((size_t)(rows + 1) * 4 + 255) & ~size_t(255);
    const size_t ib = ((size_t)std::max<int64_t>(nnz, 1) * 4 + 255) & ~size_t(255);
    char* mem = nullptr;
    cudaError_t e = cudaMalloc(&mem, pb + 2 * ib + 256);
    if (e == cudaSuccess) {
        h->row_ptr = reinterpret_cast<int32_t*>(mem);
        h->col_idx = reinterpret_cast<int32_t*>(mem + pb);
        h->vals = reinterpret_cast<float*>(mem + pb + ib);
        if (exact64) e = cudaMalloc(&h->vals64, (size_t)std::max<int64_t>(nnz, 1) * 8);
    }
    if (e != cudaSuccess) {
        spconv_csr_free(h);
        return cuda_fail(e, "cudaMalloc(matrix)");
    }
    *out = h;
    return SPCONV_OK;
}

// A CSR handle returned in `layout`: CSC goes through relayout.
static int finish_layout(spconv_csr* h, int layout, void* stream, spconv_csr** out) {
    if (layout == 0) {
        *out = h;
        return SPCONV_OK;
    }
    const int rc = spconv_relayout(h, 1, stream, out);
    const std::string msg = rc ? g_err : std::string();
    spconv_csr_free(h);
    return rc ? fail(rc, msg) : SPCONV_OK;
}

int spconv_spgemm(const spconv_csr* a, const spconv_csr* b, int layout, void* stream, spconv_csr** out) {
    if (!a || !b || !out) return fail(SPCONV_EINVAL, "spconv_spgemm: null argument");
    *out = nullptr;
    if (layout != 0 && layout != 1) return fail(SPCONV_EINVAL, "spconv_spgemm: layout must be 0 (csr) or 1 (csc)");
    if (a->cols != b->rows)
        return fail(SPCONV_EINVAL, "spgemm: inner dimensions differ, " + std::to_string(a->cols) + " vs " +
                                       std::to_string(b->rows));
    if (a->device != b->device) return fail(SPCONV_EINVAL, "spconv_spgemm: operands on different devices");
    if ((unsigned long long)a->rows * (unsigned long long)b->cols >= (1ull << 62))
        return fail(SPCONV_EINVAL, "spconv_spgemm: result too large");
    DeviceGuard dg(a->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CK(cudaDeviceSynchronize());  // the operands' builds are complete
    // Gustavson runs over rows: a conv transform held only in CSC gets a
    // row-major twin for the duration of the call (rebuilt from its taps).
    spconv_csr *ta = nullptr, *tb = nullptr;
    if (csc_native(a)) {
        if (int rc = spconv_relayout(a, 0, stream, &ta)) return rc;
        a = ta;
    }
    if (csc_native(b)) {
        if (int rc = spconv_relayout(b, 0, stream, &tb)) {
            spconv_csr_free(ta);
            return rc;
        }
        b = tb;
    }
    struct Twins {
        spconv_csr *a, *b;
        ~Twins() { spconv_csr_free(a), spconv_csr_free(b); }
    } twins{ta, tb};
    CK(cudaStreamSynchronize(st));
    spb::SpgemmIn A{a->rows, a->cols, a->nnz, a->row_ptr, a->col_idx, a->vals, a->vals64};
    spb::SpgemmIn B{b->rows, b->cols, b->nnz, b->row_ptr, b->col_idx, b->vals, b->vals64};
    spb::SpgemmOut o{};
    cudaError_t e = spb::spgemm_device(A, B, &o, st);
    if (e == cudaErrorInvalidValue) return fail(SPCONV_EINVAL, "spconv_spgemm: more than 2^31 partial products");
    CK(e);
    bool inexact = false;
    e = spb::spgemm_inexact(o, &inexact, st);
    spconv_csr* h = nullptr;
    int rc = e == cudaSuccess ? SPCONV_OK : cuda_fail(e, "spconv_spgemm");
    if (rc == SPCONV_OK && o.nnz >= (1ll << 31)) rc = fail(SPCONV_EINVAL, "spconv_spgemm: result exceeds int32");
    if (rc == SPCONV_OK) rc = new_generic(a->rows, b->cols, o.nnz, inexact, a->device, &h);
    if (rc == SPCONV_OK) {
        int maxlen = 0;
        e = spb::spgemm_finish(o, a->rows, b->cols, h->row_ptr, h->col_idx, h->vals, h->vals64, &maxlen, st);
        h->k2max = maxlen;
        if (e != cudaSuccess) {
            spconv_csr_free(h);
            rc = cuda_fail(e, "spconv_spgemm");
        }
    }
    if (o.mem) cudaFreeAsync(o.mem, st);
    cudaStreamSynchronize(st);
    if (rc != SPCONV_OK) return rc;
    return finish_layout(h, layout, stream, out);
}

int spconv_build_padding_matrix(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int layout, int device,
                                void* stream, spconv_csr** out) {
    if (!out) return fail(SPCONV_EINVAL, "spconv_build_padding_matrix: null argument");
    *out = nullptr;
    if (int rc = check_spec(m, n, k, s, p)) return rc;
    if (layout != 0 && layout != 1) return fail(SPCONV_EINVAL, "spconv_build_padding_matrix: layout must be 0 or 1");
    const int64_t rows = (m + 2 * p) * (n + 2 * p);
    if (rows >= (1ll << 31)) return fail(SPCONV_EINVAL, "spconv_build_padding_matrix: exceeds the int32 range");
    DeviceGuard dg(device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    spconv_csr* h = nullptr;
    if (int rc = new_generic(rows, m * n, m * n, false, device, &h)) return rc;
    h->k2max = 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = spb::launch_padding_matrix((int)m, (int)n, (int)p, rows, h->row_ptr, h->col_idx, h->vals, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        spconv_csr_free(h);
        return cuda_fail(e, "spconv_build_padding_matrix");
    }
    return finish_layout(h, layout, stream, out);
}

int spconv_build_conv_matrix(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, const double* kernel_kxk,
                             int layout, int device, void* stream, spconv_csr** out) {
    if (!out || !kernel_kxk) return fail(SPCONV_EINVAL, "spconv_build_conv_matrix: null argument");
    *out = nullptr;
    if (int rc = check_spec(m, n, k, s, p)) return rc;
    if (layout != 0 && layout != 1) return fail(SPCONV_EINVAL, "spconv_build_conv_matrix: layout must be 0 or 1");
    const Geom g = make_geom(m, n, k, s, p);
    const int64_t rows = g.mo * g.no, cols = (m + 2 * p) * (n + 2 * p);
    if (cols >= (1ll << 31) || rows * k * k >= (1ll << 31))
        return fail(SPCONV_EINVAL, "spconv_build_conv_matrix: exceeds the int32 range");
    std::vector<float> t32((size_t)(k * k));
    bool exact = true;
    for (int64_t q = 0; q < k * k; ++q) {
        t32[(size_t)q] = (float)kernel_kxk[q];
        exact &= __builtin_bit_cast(uint64_t, (double)t32[(size_t)q]) == __builtin_bit_cast(uint64_t, kernel_kxk[q]);
    }
    DeviceGuard dg(device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    spconv_csr* h = nullptr;
    if (int rc = new_generic(rows, cols, rows * k * k, !exact, device, &h)) return rc;
    h->k2max = (int)(k * k);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* tt = nullptr;
    cudaError_t e = cudaMallocAsync(&tt, (size_t)(k * k) * 12 + 256, st);
    float* d32 = reinterpret_cast<float*>(tt);
    double* d64 = reinterpret_cast<double*>(tt + (((size_t)(k * k) * 4 + 255) & ~size_t(255)));
    if (e == cudaSuccess) e = cudaMemcpyAsync(d32, t32.data(), (size_t)(k * k) * 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d64, kernel_kxk, (size_t)(k * k) * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = spb::launch_conv_matrix((int)k, (int)s, (int)p, (int)n, (int)g.no, rows, d32, d64, h->row_ptr,
                                    h->col_idx, h->vals, h->vals64, st);
    if (tt) cudaFreeAsync(tt, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        spconv_csr_free(h);
        return cuda_fail(e, "spconv_build_conv_matrix");
    }
    return finish_layout(h, layout, stream, out);
}

int spconv_csr_shape(const spconv_csr* h, int64_t* rows, int64_t* cols, int64_t* nnz) {
    if (!h) return fail(SPCONV_EINVAL, "null handle");
    if (rows) *rows = h->rows;
    if (cols) *cols = h->cols;
    if (nnz) *nnz = h->nnz;
    return SPCONV_OK;
}

int spconv_csr_spec(const spconv_csr* h, int64_t spec5[5]) {
    if (!h || !spec5) return fail(SPCONV_EINVAL, "null argument");
    if (h->g.m <= 0) return fail(SPCONV_EINVAL, "spconv_csr_spec: handle has no convolution geometry");
    spec5[0] = h->g.m;
    spec5[1] = h->g.n;
    spec5[2] = h->g.k;
    spec5[3] = h->g.s;
    spec5[4] = h->g.p;
    return SPCONV_OK;
}

int spconv_csr_device_ptrs(const spconv_csr* h, const int32_t** row_ptr, const int32_t** col_idx,
                           const float** vals) {
    if (!h) return fail(SPCONV_EINVAL, "null handle");
    // Writable storage leaves the library's control: a CSC conv handle is
    // checked before every later apply, which then follows the storage as it
    // stands (row-major handles re-check every call anyway: the band check).
    const_cast<spconv_csr*>(h)->exposed.store(true);
    if (row_ptr) *row_ptr = h->layout ? h->csc_ptr : h->row_ptr;
    if (col_idx) *col_idx = h->layout ? h->csc_idx : h->col_idx;
    if (vals) *vals = h->layout ? h->csc_vals : h->vals;
    return SPCONV_OK;
}

int spconv_csr_storage_bytes(const spconv_csr* h, int64_t* bytes) {
    if (!h || !bytes) return fail(SPCONV_EINVAL, "spconv_csr_storage_bytes: null argument");
    int64_t b = 0;
    if (h->row_ptr) b += 4 * (h->rows + 1) + 8 * h->nnz;
    if (h->vals64) b += 8 * h->nnz;
    if (h->csc_ptr) b += 4 * (h->cols + 1) + 8 * h->nnz;
    if (h->csc_vals64) b += 8 * h->nnz;
    *bytes = b;
    return SPCONV_OK;
}

int spconv_csr_export(const spconv_csr* h, int64_t* row_ptr, int64_t* col_idx, double* vals) {
    if (!h) return fail(SPCONV_EINVAL, "null handle");
    DeviceGuard dg(h->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    CK(cudaDeviceSynchronize());
    const int64_t major = h->layout ? h->cols : h->rows;
    if (row_ptr) {
        std::vector<int32_t> tmp((size_t)major + 1);
        CK(cudaMemcpy(tmp.data(), h->layout ? h->csc_ptr : h->row_ptr, tmp.size() * 4, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < tmp.size(); ++i) row_ptr[i] = tmp[i];
    }
    if (col_idx && h->nnz > 0) {
        std::vector<int32_t> tmp((size_t)h->nnz);
        CK(cudaMemcpy(tmp.data(), h->layout ? h->csc_idx : h->col_idx, tmp.size() * 4, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < tmp.size(); ++i) col_idx[i] = tmp[i];
    }
    const double* v64 = h->layout ? h->csc_vals64 : h->vals64;
    if (vals && h->nnz > 0 && v64) {
        CK(cudaMemcpy(vals, v64, (size_t)h->nnz * 8, cudaMemcpyDeviceToHost));
    } else if (vals && h->nnz > 0) {
        std::vector<float> tmp((size_t)h->nnz);
        CK(cudaMemcpy(tmp.data(), h->layout ? h->csc_vals : h->vals, tmp.size() * 4, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < tmp.size(); ++i) vals[i] = tmp[i];
    }
    return SPCONV_OK;
}

int spconv_csr_copy(const spconv_csr* h, int32_t* row_ptr, int32_t* col_idx, float* vals,
                    void* stream) {
    if (!h) return fail(SPCONV_EINVAL, "null handle");
    DeviceGuard dg(h->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool csc = h->layout == 1;
    if (row_ptr)
        CK(cudaMemcpyAsync(row_ptr, csc ? h->csc_ptr : h->row_ptr, (size_t)((csc ? h->cols : h->rows) + 1) * 4,
                           cudaMemcpyDefault, st));
    if (col_idx && h->nnz > 0)
        CK(cudaMemcpyAsync(col_idx, csc ? h->csc_idx : h->col_idx, (size_t)h->nnz * 4, cudaMemcpyDefault, st));
    if (vals && h->nnz > 0)
        CK(cudaMemcpyAsync(vals, csc ? h->csc_vals : h->vals, (size_t)h->nnz * 4, cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
    return SPCONV_OK;
}

// [a, a + na) and [b, b + nb) floats overlap (in-place application is not supported:
// every kernel reads x while others write y).
static bool overlaps(const float* a, int64_t na, const float* b, int64_t nb) {
    return na > 0 && nb > 0 && a < b + nb && b < a + na;
}

int spconv_spmv(const spconv_csr* h, const float* x_dev, float* y_dev, void* stream) {
    if (!h || !x_dev || !y_dev) return fail(SPCONV_EINVAL, "spconv_spmv: null argument");
    if (overlaps(x_dev, h->cols, y_dev, h->rows)) return fail(SPCONV_EINVAL, "spconv_spmv: x and y overlap");
    DeviceGuard dg(h->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    return run_spmm(const_cast<spconv_csr*>(h), x_dev, h->cols, y_dev, h->rows, 1,
                    static_cast<cudaStream_t>(stream));
}

int spconv_spmm(const spconv_csr* h, const float* X_dev, int64_t ldx, float* Y_dev, int64_t ldy,
                int64_t batch, void* stream) {
    if (!h) return fail(SPCONV_EINVAL, "spconv_spmm: null handle");
    if (batch < 0) return fail(SPCONV_EINVAL, "spconv_spmm: negative batch");
    if (batch > 0 && (!X_dev || !Y_dev)) return fail(SPCONV_EINVAL, "spconv_spmm: null buffer");
    if (ldx < h->cols || ldy < h->rows)
        return fail(SPCONV_EINVAL, "spconv_spmm: leading dimension smaller than the matrix");
    if (batch > 0 && overlaps(X_dev, (batch - 1) * ldx + h->cols, Y_dev, (batch - 1) * ldy + h->rows))
        return fail(SPCONV_EINVAL, "spconv_spmm: X and Y overlap");
    DeviceGuard dg(h->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    return run_spmm(const_cast<spconv_csr*>(h), X_dev, ldx, Y_dev, ldy, batch,
                    static_cast<cudaStream_t>(stream));
}

int spconv_convolve_host(const spconv_csr* hc, const float* X_host, float* Y_host, int64_t batch) {
    if (!hc) return fail(SPCONV_EINVAL, "spconv_convolve_host: null handle");
    if (batch < 0) return fail(SPCONV_EINVAL, "spconv_convolve_host: negative batch");
    if (batch == 0) return SPCONV_OK;
    if (!X_host || !Y_host) return fail(SPCONV_EINVAL, "spconv_convolve_host: null buffer");
    auto* h = const_cast<spconv_csr*>(hc);  // workspace only; the matrix is untouched
    std::lock_guard<std::mutex> lk(h->ws_mu);
    DeviceGuard dg(h->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    // Chunks of ~64 MB of input, double-buffered: H2D(c+1) || spmm(c) || D2H(c-1).
    const int64_t per_img = std::max<int64_t>(h->cols, 1) * 4;
    constexpr int64_t chunk_bytes = 64ll << 20;  // (16 / 32 / 128 MB: no better, profiles/r01m)
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(batch, chunk_bytes / per_img));
    if (h->ws_chunk < chunk) {
        free_ws(h);
        for (int s = 0; s < 3; ++s) {
            CK(cudaStreamCreateWithFlags(&h->ws_stream[s], cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i)
                CK(cudaEventCreateWithFlags(&h->ws_ev[s][i], cudaEventDisableTiming));
        }
        for (int i = 0; i < 2; ++i) {
            CK(cudaMalloc(&h->ws_x[i], (size_t)(chunk * h->cols * 4)));
            CK(cudaMalloc(&h->ws_y[i], (size_t)(chunk * h->rows * 4)));
        }
        h->ws_chunk = chunk;
    }
    cudaStream_t s_in = h->ws_stream[0], s_cp = h->ws_stream[1], s_out = h->ws_stream[2];
    // the build may still be in flight on its own stream (builds only enqueue);
    // once the workspace streams wait for it, everything later is ordered after it
    if (h->built && !h->ws_built_waited) {
        for (int s = 0; s < 3; ++s) CK(cudaStreamWaitEvent(h->ws_stream[s], h->built, 0));
        h->ws_built_waited = true;
    }
    // A page-locked Y is device-addressable: single-image calls have the
    // kernel write y straight into host memory (posted PCIe writes, no D2H
    // copy).  X still travels by the copy engine: reading the input windows
    // over PCIe from the kernel was slower (56^2 k3: 26.5 against 16.8 us a
    // call, scripts/probe_host.py).
    cudaPointerAttributes ay{};
    const bool y_pinned = cudaPointerGetAttributes(&ay, Y_host) == cudaSuccess && ay.type == cudaMemoryTypeHost &&
                          ay.devicePointer;
    cudaGetLastError();  // (clear the query's error state for pageable pointers)
    if (y_pinned && batch <= 2) {
        CK(cudaMemcpyAsync(h->ws_x[0], X_host, (size_t)(batch * h->cols * 4), cudaMemcpyHostToDevice, s_cp));
        if (int rc = run_spmm(h, h->ws_x[0], h->cols, static_cast<float*>(ay.devicePointer), h->rows, batch, s_cp))
            return rc;
        CK(cudaStreamSynchronize(s_cp));
        return SPCONV_OK;
    }
    if (batch <= chunk) {
        // One chunk: nothing to overlap -- H2D, apply, D2H in order on one
        // stream and a single synchronisation (the latency path of small calls).
        CK(cudaMemcpyAsync(h->ws_x[0], X_host, (size_t)(batch * h->cols * 4), cudaMemcpyHostToDevice, s_cp));
        if (int rc = run_spmm(h, h->ws_x[0], h->cols, h->ws_y[0], h->rows, batch, s_cp)) return rc;
        CK(cudaMemcpyAsync(Y_host, h->ws_y[0], (size_t)(batch * h->rows * 4), cudaMemcpyDeviceToHost, s_cp));
        CK(cudaStreamSynchronize(s_cp));
        return SPCONV_OK;
    }
    cudaEvent_t* ev_in = h->ws_ev[0];
    cudaEvent_t* ev_cp = h->ws_ev[1];
    cudaEvent_t* ev_out = h->ws_ev[2];
    // Chunk sizes ramp up from 1/8 of a chunk and back down at the end: the
    // first H2D and the last D2H are the pipeline's only unoverlapped copies.
    std::vector<int64_t> sizes;
    {
        std::vector<int64_t> ramp;
        for (int64_t r = std::max<int64_t>(1, chunk / 8); r < chunk; r *= 2) ramp.push_back(r);
        int64_t rampsum = 0;
        for (int64_t r : ramp) rampsum += r;
        if (batch >= 2 * rampsum + 2 * chunk) {
            int64_t left = batch - 2 * rampsum;
            sizes = ramp;
            while (left > 0) sizes.push_back(std::min(chunk, left)), left -= chunk;
            for (auto it = ramp.rbegin(); it != ramp.rend(); ++it) sizes.push_back(*it);
        } else {
            for (int64_t left = batch; left > 0; left -= chunk) sizes.push_back(std::min(chunk, left));
        }
    }
    int c = 0;
    for (int64_t b0 = 0; c < (int)sizes.size(); b0 += sizes[(size_t)c], ++c) {
        const int i = c & 1;
        const int64_t nb = sizes[(size_t)c];
        if (c >= 2) CK(cudaStreamWaitEvent(s_in, ev_cp[i], 0));  // spmm(c-2) done reading ws_x[i]
        CK(cudaMemcpyAsync(h->ws_x[i], X_host + b0 * h->cols, (size_t)(nb * h->cols * 4),
                           cudaMemcpyHostToDevice, s_in));
        CK(cudaEventRecord(ev_in[i], s_in));
        CK(cudaStreamWaitEvent(s_cp, ev_in[i], 0));
        if (c >= 2) CK(cudaStreamWaitEvent(s_cp, ev_out[i], 0));  // D2H(c-2) done with ws_y[i]
        if (int rc = run_spmm(h, h->ws_x[i], h->cols, h->ws_y[i], h->rows, nb, s_cp)) return rc;
        CK(cudaEventRecord(ev_cp[i], s_cp));
        CK(cudaStreamWaitEvent(s_out, ev_cp[i], 0));
        CK(cudaMemcpyAsync(Y_host + b0 * h->rows, h->ws_y[i], (size_t)(nb * h->rows * 4),
                           cudaMemcpyDeviceToHost, s_out));
        CK(cudaEventRecord(ev_out[i], s_out));
    }
    CK(cudaStreamSynchronize(s_out));
    CK(cudaStreamSynchronize(s_cp));
    CK(cudaStreamSynchronize(s_in));
    return SPCONV_OK;
}

// ---- grouped apply (group.cu) ----

// Members' y ranges pairwise disjoint and disjoint from every x (x ranges may
// share memory): one sweep over the byte ranges sorted by start.
static bool group_ranges_ok(const spconv_csr* const* hs, int64_t count, const void* const* xs, void* const* ys,
                            size_t es) {
    struct R {
        const char* a;
        const char* b;
        bool out;
    };
    std::vector<R> v;
    v.reserve((size_t)(2 * count));
    for (int64_t i = 0; i < count; ++i) {
        const char* x = static_cast<const char*>(xs[i]);
        const char* y = static_cast<const char*>(ys[i]);
        if (hs[i]->cols > 0) v.push_back({x, x + es * hs[i]->cols, false});
        if (hs[i]->rows > 0) v.push_back({y, y + es * hs[i]->rows, true});
    }
    std::sort(v.begin(), v.end(), [](const R& p, const R& q) { return p.a < q.a; });
    const char* yend = nullptr;
    const char* xend = nullptr;
    for (const R& r : v) {
        if (r.out) {
            if ((yend && r.a < yend) || (xend && r.a < xend)) return false;
            if (!yend || r.b > yend) yend = r.b;
        } else {
            if (yend && r.a < yend) return false;
            if (!xend || r.b > xend) xend = r.b;
        }
    }
    return true;
}

static int group_check(const char* who, const spconv_csr* const* hs, int64_t count, const void* const* xs,
                       void* const* ys, int* device) {
    if (count < 0) return fail(SPCONV_EINVAL, std::string(who) + ": negative count");
    if (count > 0 && (!hs || !xs || !ys)) return fail(SPCONV_EINVAL, std::string(who) + ": null array");
    for (int64_t i = 0; i < count; ++i) {
        if (!hs[i]) return fail(SPCONV_EINVAL, std::string(who) + ": null handle");
        if ((hs[i]->cols > 0 && !xs[i]) || (hs[i]->rows > 0 && !ys[i]))
            return fail(SPCONV_EINVAL, std::string(who) + ": null buffer");
        if (hs[i]->device != hs[0]->device) return fail(SPCONV_EINVAL, std::string(who) + ": handles on different devices");
        if (hs[i]->rows > INT32_MAX) return fail(SPCONV_EINVAL, std::string(who) + ": matrix too large");
    }
    *device = count > 0 ? hs[0]->device : 0;
    return SPCONV_OK;
}

// Enqueue the group on `st`: CSR members in launches of up to kGroupMax, the
// others one apply each (fp32: spconv_spmv's path; fp64: spconv_spmm_f64's).
static int run_group(const spconv_csr* const* hs, int64_t count, const void* const* xs, void* const* ys, bool f64,
                     cudaStream_t st) {
    spb::GroupParams gp;
    gp.count = 0;
    int blocks = 0;
    auto flush = [&]() -> int {
        if (gp.count > 0) CK(spb::launch_spmv_group(gp, blocks, f64, st));
        gp.count = 0;
        blocks = 0;
        return SPCONV_OK;
    };
    for (int64_t i = 0; i < count; ++i) {
        auto* h = const_cast<spconv_csr*>(hs[i]);
        if (h->rows == 0) continue;
        if (!h->row_ptr) {  // CSC-only storage: its own apply
            if (int rc = f64 ? spconv_spmm_f64(h, static_cast<const double*>(xs[i]), h->cols,
                                               static_cast<double*>(ys[i]), h->rows, 1, st)
                             : run_spmm(h, static_cast<const float*>(xs[i]), h->cols, static_cast<float*>(ys[i]),
                                        h->rows, 1, st))
                return rc;
            continue;
        }
        const bool quad = h->k2max > 16;
        const int nb = spb::group_blocks(h->rows, quad);
        if (gp.count == spb::kGroupMax || (int64_t)blocks + nb > INT32_MAX / 2)
            if (int rc = flush()) return rc;
        gp.m[gp.count++] = {h->row_ptr, h->col_idx, h->vals, f64 ? h->vals64 : nullptr, xs[i], ys[i],
                            (int)h->rows, blocks, quad ? 1 : 0};
        blocks += nb;
        h->last_kernel.store(f64 ? "csr_spmv_group<f64>" : "csr_spmv_group");
    }
    return flush();
}

static int spmv_group_impl(const char* who, const spconv_csr* const* hs, int64_t count, const void* const* xs,
                           void* const* ys, bool f64, void* stream) {
    int dev = 0;
    if (int rc = group_check(who, hs, count, xs, ys, &dev)) return rc;
    if (count == 0) return SPCONV_OK;
    if (!group_ranges_ok(hs, count, xs, ys, f64 ? 8 : 4))
        return fail(SPCONV_EINVAL, std::string(who) + ": a y overlaps another member's x or y");
    DeviceGuard dg(dev);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    return run_group(hs, count, xs, ys, f64, static_cast<cudaStream_t>(stream));
}

int spconv_spmv_group(const spconv_csr* const* hs, int64_t count, const float* const* x_dev, float* const* y_dev,
                      void* stream) {
    return spmv_group_impl("spconv_spmv_group", hs, count, reinterpret_cast<const void* const*>(x_dev),
                           reinterpret_cast<void* const*>(y_dev), false, stream);
}

int spconv_spmv_group_f64(const spconv_csr* const* hs, int64_t count, const double* const* x_dev,
                          double* const* y_dev, void* stream) {
    return spmv_group_impl("spconv_spmv_group_f64", hs, count, reinterpret_cast<const void* const*>(x_dev),
                           reinterpret_cast<void* const*>(y_dev), true, stream);
}

namespace {
// Per-device staging of spconv_convolve_host_group(_f64) (grown on demand, kept).
struct GroupWs {
    std::mutex mu;
    cudaStream_t st = nullptr;
    char* pin_in = nullptr;
    char* pin_out = nullptr;
    char* dx = nullptr;
    char* dy = nullptr;
    size_t cap_in = 0, cap_out = 0;  // bytes
};
GroupWs g_group_ws[64];
}  // namespace

static int convolve_host_group_impl(const char* who, const spconv_csr* const* hs, int64_t count,
                                    const void* const* x_host, void* const* y_host, bool f64) {
    int dev = 0;
    if (int rc = group_check(who, hs, count, x_host, y_host, &dev)) return rc;
    if (count == 0) return SPCONV_OK;
    if (dev < 0 || dev >= 64) return fail(SPCONV_EINVAL, std::string(who) + ": device index");
    DeviceGuard dg(dev);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    const size_t es = f64 ? 8 : 4;
    // packed layout, members 16-byte aligned (the band / TMA paths of CSC members)
    std::vector<size_t> xo((size_t)count), yo((size_t)count);
    size_t nin = 0, nout = 0;
    for (int64_t i = 0; i < count; ++i) {
        xo[(size_t)i] = nin;
        yo[(size_t)i] = nout;
        nin += ((size_t)hs[i]->cols * es + 15) & ~size_t(15);
        nout += ((size_t)hs[i]->rows * es + 15) & ~size_t(15);
    }
    GroupWs& w = g_group_ws[dev];
    std::lock_guard<std::mutex> lk(w.mu);
    if (!w.st) CK(cudaStreamCreateWithFlags(&w.st, cudaStreamNonBlocking));
    if (w.cap_in < nin) {
        if (w.pin_in) cudaFreeHost(w.pin_in), w.pin_in = nullptr;
        if (w.dx) cudaFree(w.dx), w.dx = nullptr;
        w.cap_in = 0;
        CK(cudaHostAlloc(&w.pin_in, nin, cudaHostAllocDefault));
        CK(cudaMalloc(&w.dx, nin));
        w.cap_in = nin;
    }
    if (w.cap_out < nout) {
        if (w.pin_out) cudaFreeHost(w.pin_out), w.pin_out = nullptr;
        if (w.dy) cudaFree(w.dy), w.dy = nullptr;
        w.cap_out = 0;
        CK(cudaHostAlloc(&w.pin_out, nout, cudaHostAllocDefault));
        CK(cudaMalloc(&w.dy, nout));
        w.cap_out = nout;
    }
    // builds only enqueue: wait for those not yet seen complete
    for (int64_t i = 0; i < count; ++i) {
        auto* h = const_cast<spconv_csr*>(hs[i]);
        if (!h->built || h->build_seen.load()) continue;
        if (cudaEventQuery(h->built) == cudaSuccess) {
            h->build_seen.store(true);
            continue;
        }
        cudaGetLastError();
        CK(cudaStreamWaitEvent(w.st, h->built, 0));
    }
    for (int64_t i = 0; i < count; ++i)
        if (hs[i]->cols > 0) std::memcpy(w.pin_in + xo[(size_t)i], x_host[i], (size_t)hs[i]->cols * es);
    CK(cudaMemcpyAsync(w.dx, w.pin_in, nin, cudaMemcpyHostToDevice, w.st));
    std::vector<const void*> xs((size_t)count);
    std::vector<void*> ys((size_t)count);
    for (int64_t i = 0; i < count; ++i) xs[(size_t)i] = w.dx + xo[(size_t)i], ys[(size_t)i] = w.dy + yo[(size_t)i];
    if (int rc = run_group(hs, count, xs.data(), ys.data(), f64, w.st)) {
        cudaStreamSynchronize(w.st);
        return rc;
    }
    CK(cudaMemcpyAsync(w.pin_out, w.dy, nout, cudaMemcpyDeviceToHost, w.st));
    CK(cudaStreamSynchronize(w.st));
    for (int64_t i = 0; i < count; ++i)
        if (hs[i]->rows > 0) std::memcpy(y_host[i], w.pin_out + yo[(size_t)i], (size_t)hs[i]->rows * es);
    return SPCONV_OK;
}

int spconv_convolve_host_group(const spconv_csr* const* hs, int64_t count, const float* const* x_host,
                               float* const* y_host) {
    return convolve_host_group_impl("spconv_convolve_host_group", hs, count,
                                    reinterpret_cast<const void* const*>(x_host),
                                    reinterpret_cast<void* const*>(y_host), false);
}

int spconv_convolve_host_group_f64(const spconv_csr* const* hs, int64_t count, const double* const* x_host,
                                   double* const* y_host) {
    return convolve_host_group_impl("spconv_convolve_host_group_f64", hs, count,
                                    reinterpret_cast<const void* const*>(x_host),
                                    reinterpret_cast<void* const*>(y_host), true);
}

int spconv_spmm_f64(const spconv_csr* h, const double* X_dev, int64_t ldx, double* Y_dev, int64_t ldy,
                    int64_t batch, void* stream) {
    return spconv_spmm_f64_threads(h, X_dev, ldx, Y_dev, ldy, batch, 1, stream);
}

int spconv_spmm_f64_threads(const spconv_csr* h, const double* X_dev, int64_t ldx, double* Y_dev, int64_t ldy,
                            int64_t batch, int threads, void* stream) {
    if (!h) return fail(SPCONV_EINVAL, "spconv_spmm_f64: null handle");
    if (batch < 0) return fail(SPCONV_EINVAL, "spconv_spmm_f64: negative batch");
    if (batch == 0) return SPCONV_OK;
    if (!X_dev || !Y_dev) return fail(SPCONV_EINVAL, "spconv_spmm_f64: null buffer");
    if (batch > INT32_MAX) return fail(SPCONV_EINVAL, "spconv_spmm_f64: batch exceeds int32");
    if (ldx < h->cols || ldy < h->rows)
        return fail(SPCONV_EINVAL, "spconv_spmm_f64: leading dimension smaller than the matrix");
    const char* xa = reinterpret_cast<const char*>(X_dev);
    const char* ya = reinterpret_cast<const char*>(Y_dev);
    if (xa < ya + 8 * ((batch - 1) * ldy + h->rows) && ya < xa + 8 * ((batch - 1) * ldx + h->cols))
        return fail(SPCONV_EINVAL, "spconv_spmm_f64: X and Y overlap");
    DeviceGuard dg(h->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    // The reference cuts the major dimension into min(threads, major) chunks
    // of ceil(major / nt); only CSC sums depend on it (inc/sparse.hpp:221-258).
    int64_t chunk = 0;
    if (h->layout == 1 && threads > 1) {
        const int64_t nt = std::min<int64_t>(threads, std::max<int64_t>(h->cols, 1));
        if (nt > 1) chunk = (h->cols + nt - 1) / nt;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto* hm = const_cast<spconv_csr*>(h);
    if (int rc = csc_sticky(h, "spconv_spmm_f64")) return rc;
    const bool csc = csc_native(h);
    if (csc && h->exposed.load()) {
        bool clean = false;
        if (int rc = csc_exposed_clean(hm, st, true, &clean)) return rc;
        if (!clean) {
            hm->last_kernel.store("csc_gather<verify>+csc_repair");
            return csc_repair_apply(hm, X_dev, ldx, Y_dev, ldy, batch, st, true, chunk);
        }
    }
    // Batches of the band geometries: the band check (CSR or CSC storage)
    // and the register-blocked apply in fp64 (spmm_band.cu, T = double) --
    // the reference's per-entry multiply and add, in its order.
    const Geom& g = h->g;
    if (chunk == 0 && batch >= 3 && h->is_conv && h->band_tw > 0 && spb::band64_supported((int)g.k, (int)g.s) &&
        (h->row_ptr || csc) && band_taps_ok(h) && path_override() != kGeneric) {
        const int sms = device_sm_count();
        spb::BandParams bp;
        spb::BandShape sh;
        if (int rc = band_setup(hm, csc, true, batch, X_dev, ldx, Y_dev, ldy, bp, sh, sms, st)) return rc;
        bp.fused = 0;
        bp.pdl = hm->applied.exchange(true) && !hm->exposed.load() && spb::opt(spb::kOptPdl) != 1 ? 1 : 0;
        CUtensorMap tmap;
        std::memset(&tmap, 0, sizeof tmap);
        RepitchBuf rbuf;
        if (int rc = repitch_for_tma(h, X_dev, ldx, batch, true, bp, sh, &tmap, rbuf, st)) return rc;
        if (!bp.notma && !rbuf.p)
            if (int rc = encode_x_map(&tmap, X_dev, g, ldx, batch, sh.wc, sh.wr, 1, true)) return rc;
        hm->checked.store(true);
        CK(spb::launch_band_check((int)g.k, (int)g.s, bp, st, sms));
        CK(spb::launch_band64((int)g.k, (int)g.s, bp, &tmap, st, nullptr, sms));
        hm->last_kernel.store(csc ? "conv_band_check<csc>+conv_spmm_band<f64>" : "conv_band_check+conv_spmm_band<f64>");
        return SPCONV_OK;
    }
    if (csc) {
        spb::CscGatherParams cp = csc_params(h, true);
        cp.X = X_dev;
        cp.ldx = ldx;
        cp.Y = Y_dev;
        cp.ldy = ldy;
        cp.batch = (int)batch;
        cp.chunk = chunk;
        CK(spb::launch_csc_gather(cp, true, st, device_sm_count()));
        hm->last_kernel.store("csc_gather<f64>");
        return SPCONV_OK;
    }
    spb::F64Params fp{h->row_ptr, h->col_idx, h->vals, h->vals64, X_dev, ldx, Y_dev, ldy, (int)h->rows, (int)batch};
    // (a CSC matrix from the host applies through its row-major arrays: the
    // row-major order of entries is the column order within each row)
    fp.chunk = chunk;
    CK(spb::launch_spmm_f64(fp, st));
    hm->last_kernel.store("csr_spmm_f64");
    return SPCONV_OK;
}

int spconv_convolve_host_f64(const spconv_csr* hc, const double* X_host, double* Y_host,
                             int64_t batch) {
    return spconv_convolve_host_f64_threads(hc, X_host, Y_host, batch, 1);
}

int spconv_convolve_host_f64_threads(const spconv_csr* hc, const double* X_host, double* Y_host,
                                     int64_t batch, int threads) {
    if (!hc) return fail(SPCONV_EINVAL, "spconv_convolve_host_f64: null handle");
    if (batch < 0) return fail(SPCONV_EINVAL, "spconv_convolve_host_f64: negative batch");
    if (batch == 0) return SPCONV_OK;
    if (!X_host || !Y_host) return fail(SPCONV_EINVAL, "spconv_convolve_host_f64: null buffer");
    // The reference-semantics path (the drop-in convolve / spmv): fp64 in,
    // fp64 arithmetic on the device (csr_spmm_f64), fp64 out.
    auto* h = const_cast<spconv_csr*>(hc);
    std::lock_guard<std::mutex> lk(h->ws_mu);
    DeviceGuard dg(h->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    keep_pool_memory(h->device);
    if (!h->ws_stream[1]) CK(cudaStreamCreateWithFlags(&h->ws_stream[1], cudaStreamNonBlocking));
    cudaStream_t st = h->ws_stream[1];
    if (h->built) CK(cudaStreamWaitEvent(st, h->built, 0));  // (builds only enqueue)
    const size_t xb = (size_t)(batch * h->cols) * 8, yb = (size_t)(batch * h->rows) * 8;
    char* buf = nullptr;
    CK(cudaMallocAsync(&buf, xb + yb, st));
    cudaError_t e = cudaMemcpyAsync(buf, X_host, xb, cudaMemcpyHostToDevice, st);
    int rc = SPCONV_OK;
    if (e == cudaSuccess)
        rc = spconv_spmm_f64_threads(h, reinterpret_cast<const double*>(buf), h->cols,
                                     reinterpret_cast<double*>(buf + xb), h->rows, batch, threads, st);
    if (e == cudaSuccess && rc == SPCONV_OK) e = cudaMemcpyAsync(Y_host, buf + xb, yb, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(buf, st);
    const cudaError_t es = cudaStreamSynchronize(st);
    if (rc != SPCONV_OK) return rc;
    if (e == cudaSuccess) e = es;
    if (e != cudaSuccess) return cuda_fail(e, "spconv_convolve_host_f64");
    return SPCONV_OK;
}

int spconv_csr_write_text(const spconv_csr* h, int transform_header_line, char* buf, int64_t cap,
                          int64_t* len) {
    if (!h || !len) return fail(SPCONV_EINVAL, "spconv_csr_write_text: null argument");
    if (transform_header_line && h->g.m <= 0)
        return fail(SPCONV_EINVAL, "write_transform: matrix has no convolution geometry");
    DeviceGuard dg(h->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    const std::string head = transform_header_line ? transform_header(h) : sparse_header(h);
    // storage order (inc/sparse.hpp:133-149): rows for CSR, columns for CSC
    const bool csc = h->layout == 1;
    const int32_t* sp_ = csc ? h->csc_ptr : h->row_ptr;
    const int32_t* si_ = csc ? h->csc_idx : h->col_idx;
    const float* sv_ = csc ? h->csc_vals : h->vals;
    const double* sv64 = csc ? h->csc_vals64 : h->vals64;
    const int64_t major = csc ? h->cols : h->rows;
    const int64_t blocks = (major + spb::text_rows_per_block() - 1) / spb::text_rows_per_block();
    CK(cudaDeviceSynchronize());  // the build (any stream) is complete
    cudaStream_t st = nullptr;
    unsigned long long* scratch = nullptr;
    CK(cudaMallocAsync(&scratch, (size_t)(blocks + 2) * 8, st));
    unsigned long long total = 0;
    cudaError_t e = spb::render_entries(sp_, si_, sv_, sv64, (int)major, scratch, nullptr, head.size(), st, true, csc);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&total, scratch + blocks, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFreeAsync(scratch, st);
        return cuda_fail(e, "spconv_csr_write_text (size)");
    }
    *len = (int64_t)total;
    if (!buf) {
        cudaFreeAsync(scratch, st);
        return SPCONV_OK;
    }
    if (cap < (int64_t)total) {
        cudaFreeAsync(scratch, st);
        return fail(SPCONV_EINVAL, "spconv_csr_write_text: buffer of " + std::to_string(cap) +
                                       " bytes is smaller than the " + std::to_string(total) + "-byte text");
    }
    char* text = nullptr;
    e = cudaMallocAsync(&text, (size_t)total + 16, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(text, head.data(), head.size(), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = spb::render_entries(sp_, si_, sv_, sv64, (int)major, scratch, text, head.size(), st, false, csc);
    if (e == cudaSuccess) e = cudaMemcpyAsync(buf, text, (size_t)total, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFreeAsync(text, st);
    cudaFreeAsync(scratch, st);
    if (e != cudaSuccess) return cuda_fail(e, "spconv_csr_write_text");
    return SPCONV_OK;
}

int spconv_sparse_read(const char* text, int64_t len, int layout, int device, void* stream, spconv_csr** out) {
    if (!text || !out || len < 0) return fail(SPCONV_EINVAL, "spconv_sparse_read: null argument");
    if (layout != 0 && layout != 1) return fail(SPCONV_EINVAL, "spconv_sparse_read: layout must be 0 (csr) or 1 (csc)");
    *out = nullptr;
    TokenReader R{text, text + len};
    int64_t rows, cols;
    std::vector<int64_t> ptr, idx;
    std::vector<double> val;
    if (int rc = parse_sparse(R, layout == 1, rows, cols, ptr, idx, val)) return rc;
    if (layout == 0) return spconv_csr_from_host(rows, cols, ptr.data(), idx.data(), val.data(), device, stream, out);
    std::vector<int32_t> cp, ci;
    std::vector<double> cv;
    transpose_host(rows, cols, ptr.data(), idx.data(), val.data(), cp, ci, cv);
    std::vector<int64_t> cp64(cp.begin(), cp.end()), ci64(ci.begin(), ci.end());
    return spconv_matrix_from_host(rows, cols, 1, cp64.data(), ci64.data(), cv.data(), device, stream, out);
}

int spconv_transform_read(const char* text, int64_t len, int device, void* stream, spconv_csr** out) {
    if (!text || !out || len < 0) return fail(SPCONV_EINVAL, "spconv_transform_read: null argument");
    *out = nullptr;
    TokenReader R{text, text + len};
    // header: "%%transform m n k s p layout" (inc/conv.hpp:226-233)
    std::string_view tag, lay;
    int64_t m, n, k, s, p;
    if (!R.next(tag) || !R.i64(m) || !R.i64(n) || !R.i64(k) || !R.i64(s) || !R.i64(p) || !R.next(lay) ||
        tag != "%%transform")
        return fail(SPCONV_ERUNTIME, "read_transform: bad header line");
    R.skip_line();
    if (int rc = check_spec(m, n, k, s, p)) return rc;
    const std::string layout(lay);
    if (layout != "csr" && layout != "CSR" && layout != "csc" && layout != "CSC")
        return fail(SPCONV_EINVAL, "unknown layout '" + layout + "' (expected csr or csc)");
    const bool csc = layout == "csc" || layout == "CSC";
    int64_t rows, cols;
    std::vector<int64_t> ptr, idx;
    std::vector<double> val;
    if (int rc = parse_sparse(R, csc, rows, cols, ptr, idx, val)) return rc;
    const int64_t nnz = (int64_t)val.size();
    const Geom g = make_geom(m, n, k, s, p);
    if (rows != g.mo * g.no || cols != m * n)
        return fail(SPCONV_ERUNTIME, "read_transform: matrix is " + std::to_string(rows) + "x" + std::to_string(cols) +
                                         " but spec " + spec_str(m, n, k, s, p) + " requires " +
                                         std::to_string(g.mo * g.no) + "x" + std::to_string(m * n));
    // If the matrix IS the conv transform of its own taps (the taps of the
    // first row that stores all k*k of them), rebuild it on the device and
    // keep the built handle: identical arrays, plus the geometry the band
    // kernels need.  Otherwise keep the upload as a generic CSR.
    std::vector<double> taps;
    for (int64_t r = 0; r < rows && taps.empty(); ++r)
        if (ptr[(size_t)r + 1] - ptr[(size_t)r] == k * k)
            for (int64_t q = 0; q < k * k; ++q) taps.push_back(val[(size_t)(ptr[(size_t)r] + q)]);
    if (!taps.empty()) {
        spconv_csr* built = nullptr;
        if (spconv_build_transform_f64(m, n, k, s, p, taps.data(), csc ? 1 : 0, device, stream, &built) ==
            SPCONV_OK) {
            bool same = built->nnz == nnz;
            if (same) {  // the storage (exact values) must equal the file's, in the file's layout
                const int64_t major = csc ? cols : rows;
                std::vector<int64_t> brp((size_t)major + 1), bci((size_t)std::max<int64_t>(nnz, 1));
                std::vector<double> bv((size_t)std::max<int64_t>(nnz, 1));
                same = spconv_csr_export(built, brp.data(), bci.data(), bv.data()) == SPCONV_OK;
                std::vector<int32_t> fcp, fci;
                std::vector<double> fcv;
                if (same && csc) transpose_host(rows, cols, ptr.data(), idx.data(), val.data(), fcp, fci, fcv);
                for (int64_t r = 0; same && r <= major; ++r)
                    same = brp[(size_t)r] == (csc ? (int64_t)fcp[(size_t)r] : ptr[(size_t)r]);
                for (int64_t e = 0; same && e < nnz; ++e)
                    same = bci[(size_t)e] == (csc ? (int64_t)fci[(size_t)e] : idx[(size_t)e]) &&
                           __builtin_bit_cast(uint64_t, bv[(size_t)e]) ==
                               __builtin_bit_cast(uint64_t, csc ? fcv[(size_t)e] : val[(size_t)e]);
            }
            if (same) {
                *out = built;
                return SPCONV_OK;
            }
            spconv_csr_free(built);
        }
    }
    spconv_csr* h = nullptr;
    if (int rc = spconv_csr_from_host(rows, cols, ptr.data(), idx.data(), val.data(), device, stream, &h))
        return rc;
    h->g = g;  // geometry travels with the matrix (Transform::spec) even when generic
    if (csc) {
        std::vector<int32_t> cp, ci;
        std::vector<double> cv;
        transpose_host(rows, cols, ptr.data(), idx.data(), val.data(), cp, ci, cv);
        std::vector<float> cvf(cv.begin(), cv.end());
        DeviceGuard dg(device);
        if (int rc = attach_csc_host(h, cp, ci, cvf, cv.data(), static_cast<cudaStream_t>(stream))) {
            const std::string msg = g_err;
            spconv_csr_free(h);
            return fail(rc, msg);
        }
    }
    *out = h;
    return SPCONV_OK;
}

const char* spconv_csr_last_kernel(const spconv_csr* h) {
    if (!h) return "";
    const char* k = h->last_kernel.load();
    return k ? k : "";
}

int spconv_band_check_status(const spconv_csr* h, int64_t* segments, int64_t* failed) {
    if (!h || !segments || !failed) return fail(SPCONV_EINVAL, "spconv_band_check_status: null argument");
    if (!h->seg_ok || h->band_tw <= 0) return fail(SPCONV_EINVAL, "spconv_band_check_status: no band geometry");
    DeviceGuard dg(h->device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    // CSR: one segment per output row x band_tw output columns; CSC storage:
    // one per input row x s * band_tw input columns
    const int64_t segw = h->band_tw / spb::band_seg_div((int)h->g.k, (int)h->g.s);
    const int64_t n = csc_native(h) ? h->g.m * h->csc_tiles_b : h->g.mo * ((h->g.no + segw - 1) / segw);
    *segments = n;
    *failed = 0;
    if (!h->checked.load()) return SPCONV_OK;  // (no check has run: nothing failed)
    std::vector<uint8_t> v((size_t)n);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(v.data(), h->seg_ok, (size_t)n, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (uint8_t b : v) bad += b == 0;
    *segments = n;
    *failed = bad;
    return SPCONV_OK;
}

int spconv_band_check_flags(const spconv_csr* h, uint8_t* out, int64_t cap, int64_t* n) {
    if (!h || !n) return fail(SPCONV_EINVAL, "spconv_band_check_flags: null argument");
    int64_t seg = 0, bad = 0;
    if (int rc = spconv_band_check_status(h, &seg, &bad)) return rc;
    *n = seg;
    if (out) {
        if (cap < seg) return fail(SPCONV_EINVAL, "spconv_band_check_flags: buffer too small");
        if (!h->checked.load()) {
            std::memset(out, 1, (size_t)seg);
            return SPCONV_OK;
        }
        DeviceGuard dg(h->device);
        CK(cudaMemcpy(out, h->seg_ok, (size_t)seg, cudaMemcpyDeviceToHost));
    }
    return SPCONV_OK;
}

int spconv_csr_free(spconv_csr* h) {
    if (!h) return SPCONV_OK;
    {
        DeviceGuard dg(h->device);
        cudaDeviceSynchronize();
        free_ws(h);
        if (h->built) cudaEventDestroy(h->built);
        if (h->row_ptr) cudaFree(h->row_ptr);
        if (h->csc_ptr) cudaFree(h->csc_ptr);
        if (h->vals64) cudaFree(h->vals64);
        if (h->csc_vals64) cudaFree(h->csc_vals64);
        if (h->taps64) cudaFree(h->taps64);
    }
    flag_free(h->fail_flag);
    delete h;
    return SPCONV_OK;
}

}  // extern "C"
