// verify.cu -- device comparators and the device verification sweep.
//
// The reference checks its sparse path against two dense comparators
// (inc/reference.hpp): direct_conv, a four-loop sliding window over a
// zero-padded copy (:41-61), and im2col_conv, an explicit k^2 x (m_out*n_out)
// patch matrix times vec(K) (:73-136).  Both run here as CUDA kernels:
//
//   * REF arithmetic (fp64, one rounded multiply then one rounded add per tap,
//     taps in (j, i) order, padding taps included): bit-identical to the
//     reference's own functions, whose Release build does not contract
//     a*b + c (x86-64 baseline, no FMA);
//   * FMA arithmetic (fp32 fmaf, same order): the device path's contract --
//     equal bit for bit to the SpMV of T for finite inputs, because a padding
//     or zero tap adds fmaf(w, 0, acc) == acc.
//
// spconv_run_verification mirrors run_verification (inc/verify.hpp:59-169)
// on the device: the same spec grid, the same seeded inputs (the reference's
// generator, inc/rng.hpp, restated below), the CSR transform and its CSC
// relayout built and applied on the GPU, compared with the device
// comparators.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/spconv_b200.h"
#include "internal.h"

namespace spb {

namespace {

template <typename T, bool FMA>
__device__ __forceinline__ T mac(T w, T v, T acc) {
    if constexpr (FMA) {
        return fma(w, v, acc);
    } else if constexpr (sizeof(T) == 8) {
        return __dadd_rn(acc, __dmul_rn(w, v));
    } else {
        return __fadd_rn(acc, __fmul_rn(w, v));
    }
}

struct ConvGeom {
    int m, n, k, s, p, mo, no;
    long long batch;
};

// direct_conv (inc/reference.hpp:41-61): one thread per output of one image.
template <typename T, bool FMA>
__global__ void __launch_bounds__(256) direct_conv_kernel(const ConvGeom G, const T* __restrict__ taps,
                                                          const T* __restrict__ A, T* __restrict__ out,
                                                          T* __restrict__ mag) {
    const long long P = (long long)G.mo * G.no;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= P * G.batch) return;
    const long long b = q / P;
    const int t = (int)(q - b * P);
    const int x = t / G.no, y = t - x * G.no;
    const T* a = A + b * (long long)G.m * G.n;
    T acc = T(0), ms = T(0);
    for (int j = 0; j < G.k; ++j) {
        const int r = G.s * x + j - G.p;
        for (int i = 0; i < G.k; ++i) {
            const int c = G.s * y + i - G.p;
            const T v = (r >= 0 && r < G.m && c >= 0 && c < G.n) ? a[(long long)r * G.n + c] : T(0);
            const T w = taps[j * G.k + i];
            acc = mac<T, FMA>(w, v, acc);
            if (mag) ms += fabs(w * v);
        }
    }
    out[q] = acc;
    if (mag) mag[q] = ms;
}

// im2col (inc/reference.hpp:73-97): patches[b][(j*k + i) * P + t] = Apad[s*x + j][s*y + i].
template <typename T>
__global__ void __launch_bounds__(256) im2col_lower_kernel(const ConvGeom G, const T* __restrict__ A,
                                                           T* __restrict__ patches) {
    const long long P = (long long)G.mo * G.no, K2 = (long long)G.k * G.k;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= K2 * P * G.batch) return;
    const long long b = q / (K2 * P);
    const long long rt = q - b * K2 * P;
    const int r = (int)(rt / P), t = (int)(rt - (long long)r * P);
    const int j = r / G.k, i = r - j * G.k;
    const int x = t / G.no, y = t - x * G.no;
    const int rr = G.s * x + j - G.p, cc = G.s * y + i - G.p;
    const T* a = A + b * (long long)G.m * G.n;
    patches[q] = (rr >= 0 && rr < G.m && cc >= 0 && cc < G.n) ? a[(long long)rr * G.n + cc] : T(0);
}

// im2col_product (inc/reference.hpp:103-118): out[t] accumulates one patch
// row at a time, r ascending -- per output the same (j, i) order as direct_conv.
template <typename T, bool FMA>
__global__ void __launch_bounds__(256) im2col_product_kernel(const ConvGeom G, const T* __restrict__ taps,
                                                             const T* __restrict__ patches,
                                                             T* __restrict__ out) {
    const long long P = (long long)G.mo * G.no, K2 = (long long)G.k * G.k;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= P * G.batch) return;
    const long long b = q / P;
    const long long t = q - b * P;
    const T* pb = patches + b * K2 * P + t;
    T acc = T(0);
    for (long long r = 0; r < K2; ++r) acc = mac<T, FMA>(taps[r], pb[r * P], acc);
    out[q] = acc;
}

template <typename T, bool FMA>
cudaError_t run_direct(const ConvGeom& g, const void* taps, const void* A, void* out, void* mag, cudaStream_t st) {
    const long long n = (long long)g.mo * g.no * g.batch;
    if (n == 0) return cudaSuccess;
    direct_conv_kernel<T, FMA><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        g, static_cast<const T*>(taps), static_cast<const T*>(A), static_cast<T*>(out), static_cast<T*>(mag));
    return cudaGetLastError();
}

template <typename T, bool FMA>
cudaError_t run_im2col(const ConvGeom& g, const void* taps, const void* A, void* out, void* patches,
                       cudaStream_t st) {
    const long long P = (long long)g.mo * g.no, K2 = (long long)g.k * g.k;
    if (P * g.batch == 0) return cudaSuccess;
    im2col_lower_kernel<T><<<(unsigned)((K2 * P * g.batch + 255) / 256), 256, 0, st>>>(
        g, static_cast<const T*>(A), static_cast<T*>(patches));
    im2col_product_kernel<T, FMA><<<(unsigned)((P * g.batch + 255) / 256), 256, 0, st>>>(
        g, static_cast<const T*>(taps), static_cast<const T*>(patches), static_cast<T*>(out));
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_direct_conv(int dtype, int m, int n, int k, int s, int p, long long batch, const void* taps,
                               const void* A, void* out, void* mag, cudaStream_t st) {
    const ConvGeom g{m, n, k, s, p, (m + 2 * p - k) / s + 1, (n + 2 * p - k) / s + 1, batch};
    return dtype == 0 ? run_direct<float, true>(g, taps, A, out, mag, st)
                      : run_direct<double, false>(g, taps, A, out, mag, st);
}

cudaError_t launch_im2col_conv(int dtype, int m, int n, int k, int s, int p, long long batch, const void* taps,
                               const void* A, void* out, void* patches, cudaStream_t st) {
    const ConvGeom g{m, n, k, s, p, (m + 2 * p - k) / s + 1, (n + 2 * p - k) / s + 1, batch};
    return dtype == 0 ? run_im2col<float, true>(g, taps, A, out, patches, st)
                      : run_im2col<double, false>(g, taps, A, out, patches, st);
}

cudaError_t launch_im2col_lower(int dtype, int m, int n, int k, int s, int p, long long batch, const void* A,
                                void* patches, cudaStream_t st) {
    const ConvGeom g{m, n, k, s, p, (m + 2 * p - k) / s + 1, (n + 2 * p - k) / s + 1, batch};
    const long long P = (long long)g.mo * g.no, K2 = (long long)k * k, total = K2 * P * batch;
    if (total == 0) return cudaSuccess;
    if (dtype == 0)
        im2col_lower_kernel<float><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
            g, static_cast<const float*>(A), static_cast<float*>(patches));
    else
        im2col_lower_kernel<double><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
            g, static_cast<const double*>(A), static_cast<double*>(patches));
    return cudaGetLastError();
}

}  // namespace spb

// ---------------------------------------------------------------------------
// Host side: the reference's seeded generator (inc/rng.hpp:22-98) and the
// verification sweep (inc/verify.hpp:59-169) over the device path.
// ---------------------------------------------------------------------------
namespace {

uint64_t splitmix64_next(uint64_t& state) {
    state += 0x9E3779B97F4A7C15ull;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

// xoshiro256++ seeded by splitmix64, Marsaglia polar normals (two per round).
struct Normal {
    uint64_t s[4];
    bool has_spare = false;
    double spare = 0.0;
    explicit Normal(uint64_t seed) {
        for (auto& w : s) w = splitmix64_next(seed);
    }
    uint64_t next_u64() {
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
    double uniform01() { return (double)(next_u64() >> 11) * 0x1.0p-53; }
    double next() {
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        double u, v, q;
        do {
            u = 2.0 * uniform01() - 1.0;
            v = 2.0 * uniform01() - 1.0;
            q = u * u + v * v;
        } while (q >= 1.0 || q == 0.0);
        const double f = std::sqrt(-2.0 * std::log(q) / q);
        spare = v * f;
        has_spare = true;
        return u * f;
    }
};

uint64_t derive_seed(uint64_t base, uint64_t index) {
    uint64_t state = base ^ (0x9E3779B97F4A7C15ull * (index + 1));
    return splitmix64_next(state);
}

std::vector<double> normals(uint64_t seed, int64_t count) {
    Normal g(seed);
    std::vector<double> v((size_t)count);
    for (auto& x : v) x = g.next();
    return v;
}

std::string spec_str(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p) {
    return "(m=" + std::to_string(m) + ", n=" + std::to_string(n) + ", k=" + std::to_string(k) +
           ", s=" + std::to_string(s) + ", p=" + std::to_string(p) + ")";
}

std::string fmt17(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

// nnz_oracle (inc/analysis.hpp:68-89): brute-force overlap count on the padded grid.
int64_t nnz_overlap(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p) {
    const int64_t pc = n + 2 * p, mo = (m + 2 * p - k) / s + 1, no = (n + 2 * p - k) / s + 1;
    std::vector<char> mask((size_t)((m + 2 * p) * pc), 0);
    for (int64_t r = 0; r < m; ++r)
        for (int64_t c = 0; c < n; ++c) mask[(size_t)((r + p) * pc + c + p)] = 1;
    int64_t total = 0;
    for (int64_t x = 0; x < mo; ++x)
        for (int64_t y = 0; y < no; ++y)
            for (int64_t j = 0; j < k; ++j)
                for (int64_t i = 0; i < k; ++i) total += mask[(size_t)((s * x + j) * pc + s * y + i)];
    return total;
}

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

}  // namespace

extern "C" {

uint64_t spconv_derive_seed(uint64_t base, uint64_t index) { return derive_seed(base, index); }

int spconv_random_normal(uint64_t seed, int64_t count, double* out) {
    if (count < 0 || (count > 0 && !out)) return spb_fail(SPCONV_EINVAL, "spconv_random_normal: bad arguments");
    Normal g(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = g.next();
    return SPCONV_OK;
}

int spconv_direct_conv(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int dtype, const void* taps_dev,
                       const void* A_dev, void* out_dev, void* mag_dev, int64_t batch, void* stream) {
    if (int rc = spconv_spec_check(m, n, k, s, p)) return rc;
    if (dtype != 0 && dtype != 1) return spb_fail(SPCONV_EINVAL, "spconv_direct_conv: dtype must be 0 (f32) or 1 (f64)");
    if (batch < 0 || (batch > 0 && (!taps_dev || !A_dev || !out_dev)))
        return spb_fail(SPCONV_EINVAL, "spconv_direct_conv: null buffer or negative batch");
    const cudaError_t e = spb::launch_direct_conv(dtype, (int)m, (int)n, (int)k, (int)s, (int)p, batch, taps_dev,
                                                  A_dev, out_dev, mag_dev, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return spb_fail(SPCONV_ECUDA, std::string("direct_conv: ") + cudaGetErrorString(e));
    return SPCONV_OK;
}

int spconv_im2col_conv(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int dtype, const void* taps_dev,
                       const void* A_dev, void* out_dev, void* patches_dev, int64_t batch, void* stream) {
    if (int rc = spconv_spec_check(m, n, k, s, p)) return rc;
    if (dtype != 0 && dtype != 1) return spb_fail(SPCONV_EINVAL, "spconv_im2col_conv: dtype must be 0 (f32) or 1 (f64)");
    if (batch < 0 || (batch > 0 && (!taps_dev || !A_dev || !out_dev || !patches_dev)))
        return spb_fail(SPCONV_EINVAL, "spconv_im2col_conv: null buffer or negative batch");
    const cudaError_t e = spb::launch_im2col_conv(dtype, (int)m, (int)n, (int)k, (int)s, (int)p, batch, taps_dev,
                                                  A_dev, out_dev, patches_dev, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return spb_fail(SPCONV_ECUDA, std::string("im2col_conv: ") + cudaGetErrorString(e));
    return SPCONV_OK;
}

// Device-resident timing of one apply method (the layer-table bench's GPU
// column): `reps` back-to-back calls captured in one CUDA graph on a private
// stream, replayed `warmup` times untimed and `trials` times between CUDA
// events; per-call mean and SEM over the trials in microseconds.
// method 0 = spconv_spmm on `h` (batch images), 1 = fp32 im2col_conv of the
// geometry and k*k taps given (one image).
int spconv_time_apply(int method, const spconv_csr* h, int64_t batch, int64_t m, int64_t n, int64_t k, int64_t s,
                      int64_t p, const float* taps_host, int64_t reps, int64_t trials, int64_t warmup,
                      double* mean_us, double* sem_us) {
    if (!mean_us || !sem_us || reps < 1 || trials < 1 || warmup < 0 || batch < 1)
        return spb_fail(SPCONV_EINVAL, "spconv_time_apply: bad arguments");
    if (method == 0 && !h) return spb_fail(SPCONV_EINVAL, "spconv_time_apply: null handle");
    if (method == 1) {
        if (int rc = spconv_spec_check(m, n, k, s, p)) return rc;
        if (!taps_host) return spb_fail(SPCONV_EINVAL, "spconv_time_apply: null taps");
    }
    if (method != 0 && method != 1) return spb_fail(SPCONV_EINVAL, "spconv_time_apply: method must be 0 or 1");
    int64_t rows, cols;
    if (method == 0) {
        int64_t nz;
        spconv_csr_shape(h, &rows, &cols, &nz);
    } else {
        rows = ((m + 2 * p - k) / s + 1) * ((n + 2 * p - k) / s + 1);
        cols = m * n;
        batch = 1;
    }
    cudaStream_t st = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    DevBuf dx, dy, dk, dpatch;
    std::vector<double> us;
    cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = dx.reserve((size_t)(batch * cols) * 4);
    if (e == cudaSuccess) e = dy.reserve((size_t)(batch * rows) * 4);
    if (e == cudaSuccess) e = cudaMemset(dx.p, 0, (size_t)(batch * cols) * 4);
    if (e == cudaSuccess && method == 1) {
        e = dk.reserve((size_t)(k * k) * 4);
        if (e == cudaSuccess) e = dpatch.reserve((size_t)(k * k * rows) * 4);
        if (e == cudaSuccess) e = cudaMemcpy(dk.p, taps_host, (size_t)(k * k) * 4, cudaMemcpyHostToDevice);
    }
    int rc = SPCONV_OK;
    auto call = [&]() -> int {
        if (method == 0)
            return spconv_spmm(h, (const float*)dx.p, cols, (float*)dy.p, rows, batch, st);
        const cudaError_t ce = spb::launch_im2col_conv(0, (int)m, (int)n, (int)k, (int)s, (int)p, 1, dk.p, dx.p,
                                                       dy.p, dpatch.p, st);
        return ce == cudaSuccess ? SPCONV_OK : spb_fail(SPCONV_ECUDA, cudaGetErrorString(ce));
    };
    if (e == cudaSuccess) rc = call();  // first use outside the capture (attributes, workspaces)
    if (e == cudaSuccess && rc == SPCONV_OK) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess && rc == SPCONV_OK) e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess && rc == SPCONV_OK) {
        for (int64_t i = 0; i < reps && rc == SPCONV_OK; ++i) rc = call();
        const cudaError_t ec = cudaStreamEndCapture(st, &graph);
        if (e == cudaSuccess) e = ec;
    }
    if (e == cudaSuccess && rc == SPCONV_OK) e = cudaGraphInstantiate(&exec, graph, 0);
    if (e == cudaSuccess && rc == SPCONV_OK) e = cudaEventCreate(&e0);
    if (e == cudaSuccess && rc == SPCONV_OK) e = cudaEventCreate(&e1);
    for (int64_t i = 0; i < warmup && e == cudaSuccess && rc == SPCONV_OK; ++i) e = cudaGraphLaunch(exec, st);
    if (e == cudaSuccess && rc == SPCONV_OK) e = cudaStreamSynchronize(st);
    for (int64_t i = 0; i < trials && e == cudaSuccess && rc == SPCONV_OK; ++i) {
        float ms = 0.0f;
        e = cudaEventRecord(e0, st);
        if (e == cudaSuccess) e = cudaGraphLaunch(exec, st);
        if (e == cudaSuccess) e = cudaEventRecord(e1, st);
        if (e == cudaSuccess) e = cudaEventSynchronize(e1);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        us.push_back(ms * 1e3 / (double)reps);
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (st) cudaStreamDestroy(st);
    if (rc != SPCONV_OK) return rc;
    if (e != cudaSuccess) return spb_fail(SPCONV_ECUDA, std::string("spconv_time_apply: ") + cudaGetErrorString(e));
    double sum = 0.0;
    for (double v : us) sum += v;
    const double mean = sum / (double)us.size();
    double sq = 0.0;
    for (double v : us) sq += (v - mean) * (v - mean);
    *mean_us = mean;
    *sem_us = us.size() > 1 ? std::sqrt(sq / (double)(us.size() - 1)) / std::sqrt((double)us.size()) : 0.0;
    return SPCONV_OK;
}

// Host-buffer fp64 forms of the comparators (the reference's own signatures
// take host grids): device buffers for one call, the device kernels, copies
// back.  mode 0 = direct_conv, 1 = im2col_conv, 2 = the im2col lowering only
// (out = the k^2 x m_out*n_out patch matrix, row-major, inc/reference.hpp:73-97).
int spconv_reference_host(int mode, int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, const double* kernel,
                          const double* A, double* out, int device) {
    if (int rc = spconv_spec_check(m, n, k, s, p)) return rc;
    if (mode < 0 || mode > 2) return spb_fail(SPCONV_EINVAL, "spconv_reference_host: mode must be 0, 1 or 2");
    if (!A || !out || (mode != 2 && !kernel)) return spb_fail(SPCONV_EINVAL, "spconv_reference_host: null buffer");
    int prev = -1;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return spb_fail(SPCONV_ECUDA, "cudaSetDevice");
    const int64_t P = ((m + 2 * p - k) / s + 1) * ((n + 2 * p - k) / s + 1);
    const int64_t outn = mode == 2 ? k * k * P : P;
    DevBuf da, dk, dout, dpatch;
    cudaError_t e = da.reserve((size_t)(m * n) * 8);
    if (e == cudaSuccess) e = dk.reserve((size_t)(k * k) * 8);
    if (e == cudaSuccess) e = dout.reserve((size_t)outn * 8);
    if (e == cudaSuccess && mode == 1) e = dpatch.reserve((size_t)(k * k * P) * 8);
    if (e == cudaSuccess) e = cudaMemcpy(da.p, A, (size_t)(m * n) * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && mode != 2) e = cudaMemcpy(dk.p, kernel, (size_t)(k * k) * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        const int M = (int)m, N = (int)n, K = (int)k, S = (int)s, Pd = (int)p;
        if (mode == 0) e = spb::launch_direct_conv(1, M, N, K, S, Pd, 1, dk.p, da.p, dout.p, nullptr, nullptr);
        else if (mode == 1) e = spb::launch_im2col_conv(1, M, N, K, S, Pd, 1, dk.p, da.p, dout.p, dpatch.p, nullptr);
        else e = spb::launch_im2col_lower(1, M, N, K, S, Pd, 1, da.p, dout.p, nullptr);
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, dout.p, (size_t)outn * 8, cudaMemcpyDeviceToHost);
    if (prev >= 0) cudaSetDevice(prev);
    if (e != cudaSuccess) return spb_fail(SPCONV_ECUDA, std::string("spconv_reference_host: ") + cudaGetErrorString(e));
    return SPCONV_OK;
}

// The padding-matrix laws for one (m, n, p): bit 0 set when P^T P is not the
// identity, bit 1 when P vec(A) is not A zero-padded; -1 on a library error.
static int padding_laws(int64_t m, int64_t n, int64_t p, uint64_t seed, int device, cudaStream_t st) {
    const int64_t mn = m * n, pr = m + 2 * p, pc = n + 2 * p, rows = pr * pc;
    spconv_csr *pm = nullptr, *pt = nullptr, *ptp = nullptr;
    int out = -1;
    do {
        if (spconv_build_padding_matrix(m, n, 1, 1, p, 0, device, st, &pm) != SPCONV_OK) break;
        int64_t r = 0, c = 0, z = 0;
        spconv_csr_shape(pm, &r, &c, &z);
        std::vector<int64_t> ptr((size_t)r + 1), idx((size_t)std::max<int64_t>(z, 1));
        std::vector<double> val((size_t)std::max<int64_t>(z, 1));
        if (spconv_csr_export(pm, ptr.data(), idx.data(), val.data()) != SPCONV_OK) break;
        // transposed (inc/sparse.hpp:276-282): the swapped entries, compiled on the device
        std::vector<int64_t> tr((size_t)std::max<int64_t>(z, 1)), tc((size_t)std::max<int64_t>(z, 1));
        for (int64_t i = 0; i < r; ++i)
            for (int64_t e = ptr[(size_t)i]; e < ptr[(size_t)i + 1]; ++e) tr[(size_t)e] = idx[(size_t)e], tc[(size_t)e] = i;
        if (spconv_matrix_from_coo(c, r, z, tr.data(), tc.data(), val.data(), 0, device, st, &pt) != SPCONV_OK) break;
        if (spconv_spgemm(pt, pm, 0, st, &ptp) != SPCONV_OK) break;
        int64_t r2 = 0, c2 = 0, z2 = 0;
        spconv_csr_shape(ptp, &r2, &c2, &z2);
        bool identity = r2 == mn && c2 == mn && z2 == mn;
        if (identity) {
            std::vector<int64_t> p2((size_t)r2 + 1), i2((size_t)std::max<int64_t>(z2, 1));
            std::vector<double> v2((size_t)std::max<int64_t>(z2, 1));
            if (spconv_csr_export(ptp, p2.data(), i2.data(), v2.data()) != SPCONV_OK) break;
            for (int64_t i = 0; i < r2 && identity; ++i)
                for (int64_t e = p2[(size_t)i]; e < p2[(size_t)i + 1]; ++e)
                    identity &= i2[(size_t)e] == i && v2[(size_t)e] == 1.0;
        }
        // P vec(A) (random_normal_grid(m, n, seed)) against A zero-padded
        const std::vector<double> a = normals(seed, mn);
        DevBuf da, dy;
        if (da.reserve((size_t)mn * 8) != cudaSuccess || dy.reserve((size_t)rows * 8) != cudaSuccess) break;
        std::vector<double> y((size_t)rows);
        if (cudaMemcpy(da.p, a.data(), (size_t)mn * 8, cudaMemcpyHostToDevice) != cudaSuccess) break;
        if (spconv_spmm_f64(pm, (const double*)da.p, mn, (double*)dy.p, rows, 1, st) != SPCONV_OK) break;
        if (cudaMemcpy(y.data(), dy.p, (size_t)rows * 8, cudaMemcpyDeviceToHost) != cudaSuccess) break;
        bool pad_ok = true;
        for (int64_t rr = 0; rr < pr && pad_ok; ++rr)
            for (int64_t cc = 0; cc < pc && pad_ok; ++cc) {
                const bool inside = rr >= p && rr < p + m && cc >= p && cc < p + n;
                const double want = inside ? a[(size_t)((rr - p) * n + (cc - p))] : 0.0;
                pad_ok = y[(size_t)(rr * pc + cc)] == want;
            }
        out = (identity ? 0 : 1) | (pad_ok ? 0 : 2);
    } while (false);
    spconv_csr_free(ptp);
    spconv_csr_free(pt);
    spconv_csr_free(pm);
    return out;
}

int spconv_run_verification(int64_t max_dim, int seeds, uint64_t base_seed, int device, int64_t counts[4],
                            double devs[3], char* failures, int64_t cap) {
    if (!counts || !devs) return spb_fail(SPCONV_EINVAL, "spconv_run_verification: null argument");
    if (max_dim < 1 || seeds < 0) return spb_fail(SPCONV_EINVAL, "spconv_run_verification: bad options");
    int prev = -1;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return spb_fail(SPCONV_ECUDA, "cudaSetDevice");
    const double conv_tol = 1e-10;  // fp64 comparators vs each other (VerifyOptions::conv_tol)
    const double f32_tol = 1e-5;    // fp32 device path, condition-relative (BASELINE north star)
    const size_t max_failures = 20;
    int64_t specs = 0, conv_cases = 0, clipped = 0;
    double max_conv_dev = 0.0, max_rel_dev = 0.0, max_layout_dev = 0.0;
    std::vector<std::string> fails;
    auto fail = [&](const std::string& msg) {
        if (fails.size() < max_failures) fails.push_back(msg);
    };
    cudaStream_t st = nullptr;
    DevBuf b_a32, b_a64, b_a64u, b_k32, b_k64, b_k64u, b_y32c, b_y32s, b_d32, b_ref_r, b_ref, b_mag, b_i2c, b_y64c,
        b_y64s, b_patch;
    uint64_t case_index = 0;
    int rc = SPCONV_OK;
    bool stop = false;  // a CUDA error, or max_failures collected (run_verification returns early)
    for (int64_t m = 1; m <= max_dim && !stop; ++m)
        for (int64_t n = 1; n <= max_dim && !stop; ++n)
            for (int64_t p = 0; p <= 3 && !stop; ++p)
                for (int64_t s = 1; s <= 3 && !stop; ++s) {
                    const int64_t k_max = std::min(m, n) + 2 * p;
                    for (int64_t k = 1; k <= k_max && !stop; ++k) {
                        ++specs;
                        const std::string ss = spec_str(m, n, k, s, p);
                        const int64_t mo = (m + 2 * p - k) / s + 1, no = (n + 2 * p - k) / s + 1;
                        const int64_t P = mo * no, mn = m * n;
                        int64_t bound = 0;
                        spconv_nnz_bound(m, n, k, s, p, &bound);
                        const int64_t oracle = nnz_overlap(m, n, k, s, p);
                        if (bound != oracle)
                            fail("nnz_bound " + std::to_string(bound) + " != oracle " + std::to_string(oracle) +
                                 " for " + ss);
                        const int64_t dense = P * k * k;
                        if (p == 0 && bound != dense)
                            fail("p=0 bound " + std::to_string(bound) + " != dense " + std::to_string(dense) +
                                 " for " + ss);
                        if (bound < 0 || bound > dense) fail("bound outside [0, dense] for " + ss);
                        {  // clipped: some placement sees only padding (closed form, inc/analysis.hpp:21-52)
                            bool any0 = false;
                            for (int64_t x = 0; x < mo && !any0; ++x) {
                                const int64_t a = std::max<int64_t>(0, k - (std::max<int64_t>(0, p - s * x) +
                                                                           std::max<int64_t>(0, s * x + k - m - p)));
                                for (int64_t y = 0; y < no && !any0; ++y) {
                                    const int64_t c = std::max<int64_t>(0, k - (std::max<int64_t>(0, p - s * y) +
                                                                               std::max<int64_t>(0, s * y + k - n - p)));
                                    any0 = a * c == 0;
                                }
                            }
                            if (any0) ++clipped;
                        }
                        // Padding-matrix laws, which depend only on (m, n, p)
                        // (inc/verify.hpp:96-122): P built on the device, P^T by a
                        // device compile of the swapped entries, P^T P by the device
                        // spgemm -- the identity; P vec(A) by the fp64 SpMV -- A
                        // zero-padded, exactly.
                        if (k == 1 && s == 1) {
                            const uint64_t pseed = derive_seed(base_seed, case_index++);
                            const int plaw = padding_laws(m, n, p, pseed, device, st);
                            if (plaw < 0) {
                                rc = SPCONV_ECUDA;
                                stop = true;
                                break;
                            }
                            if (plaw & 1) fail("PtP != identity for " + ss);
                            if (plaw & 2) fail("P*vec(A) != zero-padded A for " + ss);
                            if (fails.size() >= max_failures) stop = true;
                        }
                        for (int sd = 0; sd < seeds && !stop; ++sd) {
                            const uint64_t cs = derive_seed(base_seed, case_index++);
                            const std::vector<double> a64 = normals(cs, mn);
                            std::vector<double> k64;
                            for (int attempt = 0;; ++attempt) {  // detail::nonzero_kernel (:47-55)
                                k64 = normals(derive_seed(cs, 7) + (uint64_t)attempt, k * k);
                                bool z = false;
                                for (double v : k64) z |= v == 0.0;
                                if (!z) break;
                            }
                            std::vector<float> a32(a64.begin(), a64.end()), k32(k64.begin(), k64.end());
                            // fp32 leg: the fp64 comparators see the fp32-rounded data it sees
                            std::vector<double> a64r(a32.begin(), a32.end()), k64r(k32.begin(), k32.end());
                            // One CSR build from the reference's double taps (exact fp64 values +
                            // the fp32-narrowed ones) and its CSC relayout serve both legs.
                            spconv_csr *tc = nullptr, *tcsc = nullptr;
                            if (spconv_build_transform_f64(m, n, k, s, p, k64.data(), 0, device, st, &tc) != SPCONV_OK ||
                                spconv_relayout(tc, 1, st, &tcsc) != SPCONV_OK) {
                                rc = SPCONV_ECUDA;
                                stop = true;
                                if (tc) spconv_csr_free(tc);
                                break;
                            }
                            int64_t rr, cc, nz;
                            spconv_csr_shape(tc, &rr, &cc, &nz);
                            if (nz != bound)
                                fail("nnz(T) " + std::to_string(nz) + " != bound " + std::to_string(bound) + " for " +
                                     ss);
                            std::vector<float> ycsr((size_t)P), ycsc((size_t)P), yd32((size_t)P);
                            std::vector<double> yref_r((size_t)P), ymag((size_t)P);
                            std::vector<double> yref((size_t)P), yi2c((size_t)P), y64c((size_t)P), y64s((size_t)P);
                            cudaError_t e = cudaSuccess;
                            auto ok = [&](cudaError_t x) { return (e = (e == cudaSuccess ? x : e)) == cudaSuccess; };
                            ok(b_a32.reserve(mn * 4));
                            ok(b_a64.reserve(mn * 8));
                            ok(b_a64u.reserve(mn * 8));
                            ok(b_k32.reserve(k * k * 4));
                            ok(b_k64.reserve(k * k * 8));
                            ok(b_k64u.reserve(k * k * 8));
                            ok(b_y32c.reserve(P * 4));
                            ok(b_y32s.reserve(P * 4));
                            ok(b_d32.reserve(P * 4));
                            ok(b_ref_r.reserve(P * 8));
                            ok(b_ref.reserve(P * 8));
                            ok(b_mag.reserve(P * 8));
                            ok(b_i2c.reserve(P * 8));
                            ok(b_y64c.reserve(P * 8));
                            ok(b_y64s.reserve(P * 8));
                            ok(b_patch.reserve(P * k * k * 8));
                            ok(cudaMemcpy(b_a32.p, a32.data(), mn * 4, cudaMemcpyHostToDevice));
                            ok(cudaMemcpy(b_a64.p, a64r.data(), mn * 8, cudaMemcpyHostToDevice));
                            ok(cudaMemcpy(b_a64u.p, a64.data(), mn * 8, cudaMemcpyHostToDevice));
                            ok(cudaMemcpy(b_k32.p, k32.data(), k * k * 4, cudaMemcpyHostToDevice));
                            ok(cudaMemcpy(b_k64.p, k64r.data(), k * k * 8, cudaMemcpyHostToDevice));
                            ok(cudaMemcpy(b_k64u.p, k64.data(), k * k * 8, cudaMemcpyHostToDevice));
                            int r1 = SPCONV_OK;
                            if (e == cudaSuccess) {
                                // fp64 leg -- the reference's own check (inc/verify.hpp:124-155)
                                r1 |= spconv_spmm_f64(tc, (const double*)b_a64u.p, mn, (double*)b_y64c.p, P, 1, st);
                                r1 |= spconv_spmm_f64(tcsc, (const double*)b_a64u.p, mn, (double*)b_y64s.p, P, 1, st);
                                r1 |= spconv_direct_conv(m, n, k, s, p, 1, b_k64u.p, b_a64u.p, b_ref.p, nullptr, 1, st);
                                r1 |= spconv_im2col_conv(m, n, k, s, p, 1, b_k64u.p, b_a64u.p, b_i2c.p, b_patch.p, 1, st);
                                // fp32 leg -- the batch kernels' contract
                                r1 |= spconv_spmv(tc, (const float*)b_a32.p, (float*)b_y32c.p, st);
                                r1 |= spconv_spmv(tcsc, (const float*)b_a32.p, (float*)b_y32s.p, st);
                                r1 |= spconv_direct_conv(m, n, k, s, p, 0, b_k32.p, b_a32.p, b_d32.p, nullptr, 1, st);
                                r1 |= spconv_direct_conv(m, n, k, s, p, 1, b_k64.p, b_a64.p, b_ref_r.p, b_mag.p, 1, st);
                            }
                            ok(cudaMemcpy(ycsr.data(), b_y32c.p, P * 4, cudaMemcpyDeviceToHost));
                            ok(cudaMemcpy(ycsc.data(), b_y32s.p, P * 4, cudaMemcpyDeviceToHost));
                            ok(cudaMemcpy(yd32.data(), b_d32.p, P * 4, cudaMemcpyDeviceToHost));
                            ok(cudaMemcpy(yref_r.data(), b_ref_r.p, P * 8, cudaMemcpyDeviceToHost));
                            ok(cudaMemcpy(ymag.data(), b_mag.p, P * 8, cudaMemcpyDeviceToHost));
                            ok(cudaMemcpy(yref.data(), b_ref.p, P * 8, cudaMemcpyDeviceToHost));
                            ok(cudaMemcpy(yi2c.data(), b_i2c.p, P * 8, cudaMemcpyDeviceToHost));
                            ok(cudaMemcpy(y64c.data(), b_y64c.p, P * 8, cudaMemcpyDeviceToHost));
                            ok(cudaMemcpy(y64s.data(), b_y64s.p, P * 8, cudaMemcpyDeviceToHost));
                            spconv_csr_free(tcsc);
                            spconv_csr_free(tc);
                            if (e != cudaSuccess || r1 != SPCONV_OK) {
                                rc = spb_fail(SPCONV_ECUDA, std::string("verification sweep: ") +
                                                                (e != cudaSuccess ? cudaGetErrorString(e)
                                                                                  : "device call failed"));
                                stop = true;
                                break;
                            }
                            ++conv_cases;
                            // fp64 leg: the reference's deviations (its report's max_conv_dev /
                            // max_layout_dev, both 0 on the reference's own grid)
                            double dev = 0.0, ldev = 0.0;
                            for (int64_t t = 0; t < P; ++t) {
                                dev = std::max(dev, std::fabs(y64c[t] - yref[t]));
                                dev = std::max(dev, std::fabs(y64s[t] - yref[t]));
                                dev = std::max(dev, std::fabs(yi2c[t] - yref[t]));
                                dev = std::max(dev, std::fabs(y64c[t] - yi2c[t]));
                                ldev = std::max(ldev, std::fabs(y64c[t] - y64s[t]));
                            }
                            max_conv_dev = std::max(max_conv_dev, dev);
                            max_layout_dev = std::max(max_layout_dev, ldev);
                            if (dev > conv_tol)
                                fail("convolution mismatch (dev " + fmt17(dev) + ") for " + ss + " seed " +
                                     std::to_string(sd));
                            if (ldev > 0.0)
                                fail("CSR/CSC mismatch (dev " + fmt17(ldev) + ") for " + ss + " seed " +
                                     std::to_string(sd));
                            // fp32 leg: bit-equal to the fp32 direct_conv, CSR == CSC, and within
                            // f32_tol * sum|w*a| of the fp64 result on the same rounded data
                            double rel = 0.0;
                            bool exact = true, same = true;
                            for (int64_t t = 0; t < P; ++t) {
                                const double d32 = std::fabs((double)ycsr[t] - yref_r[t]);
                                if (ymag[t] > 0) rel = std::max(rel, d32 / ymag[t]);
                                else if (d32 > 0) rel = INFINITY;
                                exact &= std::memcmp(&ycsr[t], &yd32[t], 4) == 0;
                                same &= std::memcmp(&ycsr[t], &ycsc[t], 4) == 0;
                            }
                            max_rel_dev = std::max(max_rel_dev, rel);
                            if (rel > f32_tol)
                                fail("fp32 convolution deviation (rel " + fmt17(rel) + ") for " + ss + " seed " +
                                     std::to_string(sd));
                            if (!exact) fail("sparse != fp32 direct_conv for " + ss + " seed " + std::to_string(sd));
                            if (!same) fail("fp32 CSR/CSC mismatch for " + ss + " seed " + std::to_string(sd));
                        }
                        if (fails.size() >= max_failures) stop = true;
                    }
                }
    if (prev >= 0) cudaSetDevice(prev);
    if (rc != SPCONV_OK) return rc;
    counts[0] = specs;
    counts[1] = conv_cases;
    counts[2] = clipped;
    counts[3] = (int64_t)fails.size();
    devs[0] = max_conv_dev;
    devs[1] = max_layout_dev;
    devs[2] = max_rel_dev;
    if (failures && cap > 0) {
        std::string all;
        for (auto& f : fails) all += f + "\n";
        const size_t nb = std::min<size_t>(all.size(), (size_t)cap - 1);
        std::memcpy(failures, all.data(), nb);
        failures[nb] = '\0';
    }
    return SPCONV_OK;
}

}  // extern "C"
