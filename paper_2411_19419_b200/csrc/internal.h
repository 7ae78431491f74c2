// internal.h -- shared host/device declarations of the B200 conv-as-SpMV library.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <vector>

namespace spb {

// Process-wide path options (options.cu, spconv_set_option): 0 = the library's
// own choice everywhere.  Values follow the symbolic lists in options.cu.
enum Opt {
    kOptPath = 0,      // 0 auto, 1 banded, 2 tiled, 3 tiled_notma, 4 generic, 5 spmv, 6 spmv_plain
    kOptFused,         // 0 auto, 1 two kernels, 2 fused check + apply
    kOptGeneric,       // 0 row-block multi-vector kernel, 1 thread per row
    kOptBuild,         // 0 auto, 1 block, 2 warp, 3 persist
    kOptBulkStoreOff,  // 0 bulk (TMA) stores of staged entries, 1 per-thread 16-byte stores
    kOptStage,         // latency SpMV: 0 auto (window kernel from 8 MB of matrix), 1 bulk-staged, 2 window
    kOptSpecSkew,      // test hook: offsets the latency SpMV's predicted row starts
    kOptRepitch,       // band path on rows not 16-byte pitched: 0 auto (repitched copy + TMA), 1 off (element staging)
    kOptPdl,           // band kernels as programmatic dependent launches: 0 auto, 1 off, 2 the apply only (check normal)
    kOptCount
};
extern std::atomic<int> g_opt[kOptCount];
inline int opt(Opt o) { return g_opt[o].load(std::memory_order_relaxed); }

// Geometry of one padded, strided convolution (inc/conv.hpp:33-62).
struct Geom {
    int64_t m, n, k, s, p;
    int64_t mo, no;  // m_out, n_out (inc/conv.hpp:52-53)
};

// Host-precomputed O(k^2) tables of the closed-form build (see csr_build.cu).
struct BuildTables {
    const float* taps;     // k*k, fp32, row-major
    const int32_t* sat;    // (k+1)*(k+1) summed-area table of (tap != 0)
    const long long* w;    // k: W[j] = sum_i nz[j][i] * #{y : i in I(y)}
};

constexpr int kSmallK = 16;  // tables travel in the kernel parameters up to this k
struct SmallTables {
    float taps[kSmallK * kSmallK];
    int32_t sat[(kSmallK + 1) * (kSmallK + 1)];
    long long w[kSmallK];
};

struct BuildParams {
    int m, n, k, s, p, mo, no;
    int rows;
    int small;        // 1: tables in `tab`, 0: tables in device memory `t`
    int stage;        // 1: stage entries in shared memory, 0: direct stores
    int stage_words;  // words per staging array
    SmallTables tab;
    BuildTables t;
    int32_t* row_ptr;
    int32_t* col_idx;
    float* vals;
    float* taps_out;  // k*k taps copied here by block 0 (the handle's device tap table)
    int bulk_store;   // write staged entries back with TMA bulk stores (else 16-byte st.global)
    long long nnz_total;  // total entries (the persistent build's last-tile bound)
    // Exact-fp64 builds (spconv_build_transform_f64): the taps above are TAGS
    // (q + 1 where the double tap is non-zero); the persistent kernel (k <= 5)
    // writes f64_t32[q] to vals and f64_t64[q] to vals64 from its staging.
    float f64_t32[121];  // (k <= 11: in the parameters, no copies)
    double f64_t64[121];
    double* vals64;
};

// CSC build (csc_build.cu): the conv transform stored column-major.
struct CscParams {
    int m, n, k, s, p, mo, no;
    int cols;
    int stage;        // 1: stage entries in shared memory
    int stage_words;  // words per staging array
    int bulk_store;   // write staged entries back with TMA bulk stores
    const float* taps;  // device k*k taps
    int32_t* col_ptr;
    int32_t* row_idx;
    float* vals;
};

// Conv-tiled SpMM: one CTA owns a TH x 32 block of output pixels (rows of T)
// and streams the whole batch through shared memory.
struct TiledParams {
    const int32_t* row_ptr;
    const int32_t* col_idx;
    const float* vals;
    const float* X;
    int64_t ldx;
    float* Y;
    int64_t ldy;
    int batch;
    int m, n, s, p, mo, no;
    int th;          // tile height (output rows of the image); tile width is 32
    int tiles_y;     // tiles across n_out
    int wr, wc;      // staged input window: rows x cols (wc % 4 == 0)
    int k2max;       // max stored entries per row of T
    int stages;      // window pipeline depth (TMA path)
    int use_tma;
};

// Two-kernel conv SpMM (spmm_band.cu): band check + register-blocked apply.
struct BandParams {
    const int32_t* row_ptr;
    const int32_t* col_idx;
    const float* vals;
    const float* taps;   // k*k fp32 taps of the handle (device)
    uint8_t* seg_ok;     // [mo][tiles_y] band-check result
    const float* X;
    int64_t ldx;
    float* Y;
    int64_t ldy;
    int batch;
    int m, n, p, mo, no;
    int tiles_y;       // tiles across n_out
    int tiles;         // tiles_x * tiles_y
    int fast_allowed;  // every tap finite and non-zero
    int y_vec;         // Y rows admit CPT-wide vector stores
    int sy;            // sum over output columns y of cy(y) (closed-form row starts)
    int nnz;
    int fused;         // host: launch the fused check + apply (+ fixup) instead of two kernels
    int zt;            // some taps are exact zeros (not stored): masked footprint + checks
    unsigned long long nzmask;  // bit j*k+i: tap (j, i) is non-zero (zt; k <= 7)
    long long zw[8];            // zt: W[j] = sum_i nz[j][i] * #{y : tap i lands} (per handle)
    // CSC storage (csc = 1): row_ptr / col_idx / vals above hold col_ptr /
    // row_idx / vals of the column-major storage, the check verifies it
    // segment by segment (one input image row x TW input columns, tiles_b
    // segments per input row) and the apply never reads it per entry.
    int csc;
    int tiles_b;
    int* fail_count;  // set to 1 when a segment fails and nothing repairs it (the handle's sticky verdict)
    int fixup;        // fused CSR form: launch conv_band_fixup for failed segments (storage handed out)
    // fp64 apply (spconv_spmm_f64; X / Y then hold doubles): the exact taps and
    // per-entry values when the handle keeps them (NULL: the fp32 ones widened)
    const double* taps64;
    const double* vals64;
    int notma;         // X rows not 16-byte pitched (or windows wider than a TMA box): cp.async staging
    int seg_div;       // check segments per apply tile width (k = 11: smaller segments)
    int tiles_y_chk;   // check segments across n_out (CSR storage) = ceil(n_out / (TW / seg_div))
    int pdl;           // host: launch the apply as a programmatic dependent of the previous kernel
};

// CSC-storage SpMV / SpMM of a conv transform (csc_apply.cu).
struct CscGatherParams {
    const int32_t* col_ptr;
    const int32_t* row_idx;
    const float* vals;
    const double* vals64;  // exact values when the handle keeps them (fp64 mode compares / applies them)
    const float* taps32;   // device k*k fp32 taps (what vals must equal)
    const double* taps64;  // device k*k exact taps (NULL: taps32 widened)
    const void* X;         // float or double, image-major
    int64_t ldx;
    void* Y;
    int64_t ldy;
    int batch;
    int m, n, k, s, p, mo, no;
    long long rows, cols, nnz;
    int zt;                   // some taps are exact zeros (not stored)
    uint32_t nzrow[32];       // bit i of nzrow[j]: tap (j, i) is stored (all ones for dense taps); k <= 32
    long long zw[32];         // W[j] = sum_i nz[j][i] * #{y : tap i lands}
    long long chunk;          // fp64: columns per reference thread (0: one thread)
    int verify_only;          // 1: check the storage, no sums
    int* fail;                // set to 1 when the storage is not the transform of the taps
    int inline_taps;          // k <= 7: the fp32 taps below (the latency kernel reads them from here)
    float it32[49];
};
cudaError_t launch_csc_gather(const CscGatherParams& cp, bool f64, cudaStream_t st, int sms);
// One or two fp32 images, k <= 7 (taps inline): loads issued a row at a time, PDL-chained.
cudaError_t launch_csc_gather_lat(const CscGatherParams& cp, cudaStream_t st, int sms, bool pdl);

// One launch over a list of CSR transforms, each applied to its own vector
// (group.cu).  Member m owns blocks [blk0, next blk0) of the grid.
struct GroupMember {
    const int32_t* row_ptr;
    const int32_t* col_idx;
    const float* vals;
    const double* vals64;  // fp64 group: the exact values when the handle keeps them
    const void* x;         // float / double
    void* y;
    int rows;
    int blk0;
    int quad;  // 1: rows of more than 16 entries, four lanes per row (group.cu)
};
constexpr int kGroupMax = 128;  // members per launch (8 KB of kernel parameters)
struct GroupParams {
    int count;
    GroupMember m[kGroupMax];
};
cudaError_t launch_spmv_group(const GroupParams& gp, int blocks, bool f64, cudaStream_t st);
// Copy of `batch` images (rows of n elements at X[b*ldx + r*n + c]) into rows of
// np >= n elements (Xp[(b*m + r)*np + c]): a 16-byte pitched layout TMA can
// describe (repitch.cu).
cudaError_t launch_repitch(const void* X, int64_t ldx, void* Xp, int m, int n, int64_t np, int64_t batch, bool f64,
                           cudaStream_t st);
int group_blocks(int64_t rows, bool quad);

struct BandShape {
    int th, tw, wr, wc, smem, threads, occ;
};

// Warp-per-32-rows latency SpMV (spmm.cu, batch <= 2).
struct SpecParams {
    const int32_t* row_ptr;
    const int32_t* col_idx;
    const float* vals;
    const float* X;
    int64_t ldx;
    float* Y;
    int64_t ldy;
    int rows, batch, nnz;
    int m, n, k, s, p, mo, no;
    int sy;    // sum over output columns y of cy(y)
    int skew;  // test hook: offsets the predicted row start (forces the mismatch path)
    int pdl;   // host: launch as a programmatic dependent of the previous kernel
    int zt;    // zero taps (k <= 7): row starts from the tap mask and W[j]
    unsigned long long nzmask;
    long long zw[8];
};

struct GenericParams {
    const int32_t* row_ptr;
    const int32_t* col_idx;
    const float* vals;
    const float* X;
    int64_t ldx;
    float* Y;
    int64_t ldy;
    int rows;
    int batch;
    int stage_cap = 0;  // csr_spmm_rowblock: staged entries per CTA (set by its launcher)
};

// Launchers (return cudaError_t of the launch).
cudaError_t launch_csr_build(const BuildParams& bp, bool dense, int block, size_t smem, bool* f64_done,
                             cudaStream_t st);
cudaError_t launch_csc_build(CscParams cp, int maxc, bool dense, cudaStream_t st);  // dense: no zero taps
cudaError_t launch_tiled(const TiledParams& tp, const CUtensorMap* tmap, int bt, size_t smem,
                         cudaStream_t st);
cudaError_t launch_generic(const GenericParams& gp, cudaStream_t st);
cudaError_t launch_rowblock(GenericParams gp, int kmax, cudaStream_t st);  // rows of <= 64 entries
// spgemm on the device (coo.cu): the operands' row-major arrays (fp64 values
// when the handle keeps them, else fp32 widened).
struct SpgemmIn {
    long long rows, cols, nnz;
    const int32_t* ptr;
    const int32_t* idx;
    const float* v32;
    const double* v64;
};
struct SpgemmOut {
    long long nnz, max_len;
    unsigned long long* keys_buf;  // sorted (row * cols + col) keys of the kept entries
    double* vals_buf;              // their sums
    void* mem;                     // owns both (cudaFreeAsync)
};
cudaError_t spgemm_device(const SpgemmIn& A, const SpgemmIn& B, SpgemmOut* out, cudaStream_t st);
cudaError_t spgemm_finish(const SpgemmOut& o, long long nrows, long long ncols, int32_t* ptr, int32_t* idx, float* v32,
                          double* v64, int* max_len, cudaStream_t st);
cudaError_t spgemm_inexact(const SpgemmOut& o, bool* inexact, cudaStream_t st);
cudaError_t launch_padding_matrix(int m, int n, int p, long long rows, int32_t* ptr, int32_t* idx, float* val,
                                  cudaStream_t st);
cudaError_t launch_conv_matrix(int k, int s, int p, int n, int no, long long rows, const float* t32,
                               const double* t64, int32_t* ptr, int32_t* idx, float* v32, double* v64,
                               cudaStream_t st);
// SparseMatrix::compile of host triplets on the device (coo.cu).
cudaError_t coo_compile(long long n, const int64_t* r_host, const int64_t* c_host, const double* v_host,
                        int64_t rows, int64_t cols, bool by_row, int32_t* ptr, int32_t* idx, float* v32,
                        double* v64, long long* dup_index, int64_t* dup_r, int64_t* dup_c, int* max_len,
                        cudaStream_t st);
struct F64Params {
    const int32_t* row_ptr;
    const int32_t* col_idx;
    const float* vals;
    const double* vals64;  // exact values when the handle keeps them (else NULL: vals widened)
    const double* X;
    int64_t ldx;
    double* Y;
    int64_t ldy;
    int rows, batch;
    long long chunk = 0;  // columns per reference thread (CSC thread-order combine; 0: one thread)
};
cudaError_t launch_spmm_f64(const F64Params& fp, cudaStream_t st);
// Tag -> value pass of the exact-fp64 build: vals[e] holds (float)(q + 1) for
// tap q; rewritten to t32[q], and vals64[e] = t64[q] (csr_build.cu).
cudaError_t launch_retag(float* vals, double* vals64, int64_t nnz, const float* t32, const double* t64,
                         cudaStream_t st);
cudaError_t launch_spmv_unrolled(const GenericParams& gp, int kmax, cudaStream_t st);
cudaError_t launch_spmv_warp(const SpecParams& sp, int kmax, bool spec, cudaStream_t st);
// One-round-trip latency SpMV of conv transforms (matrix run + input window together).
bool spmv_win_ok(const SpecParams& sp);
cudaError_t launch_spmv_win(const SpecParams& sp, int kmax, cudaStream_t st);

bool band_supported(int k, int s);
int band_tile_width(int k, int s);
int band_seg_div(int k, int s);       // check segments per tile width
int band_csc_seg_div(int k, int s);   // the same for CSC storage
bool band64_supported(int k, int s);  // fp64 apply instantiated
cudaError_t launch_band(int k, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st,
                        BandShape* shape, int sms);
cudaError_t launch_band_check(int k, int s, const BandParams& bp, cudaStream_t st, int sms);
// The same apply in fp64 (X / Y doubles; the check kernel above runs first).
cudaError_t launch_band64(int k, int s, const BandParams& bp, const CUtensorMap* tmap, cudaStream_t st,
                          BandShape* shape, int sms);

cudaError_t render_entries(const int32_t* row_ptr, const int32_t* col_idx, const float* vals,
                           const double* vals64, int rows, unsigned long long* scratch, char* out_dev, unsigned long long base,
                           cudaStream_t st, bool size_only, bool swap);
int text_rows_per_block();

size_t tiled_smem_bytes(int th, int wr, int wc, int k2max, int bt, int stages);

// Device comparators (verify.cu): dtype 0 = fp32 fmaf (the device contract),
// 1 = fp64 without contraction (bit-identical to inc/reference.hpp).
cudaError_t launch_direct_conv(int dtype, int m, int n, int k, int s, int p, long long batch, const void* taps,
                               const void* A, void* out, void* mag, cudaStream_t st);
cudaError_t launch_im2col_conv(int dtype, int m, int n, int k, int s, int p, long long batch, const void* taps,
                               const void* A, void* out, void* patches, cudaStream_t st);
cudaError_t launch_im2col_lower(int dtype, int m, int n, int k, int s, int p, long long batch, const void* A,
                                void* patches, cudaStream_t st);

}  // namespace spb

// Sets the calling thread's spconv_last_error() message and returns `code` (capi.cu).
#include <string>
int spb_fail(int code, const std::string& msg);

// The opaque handle of include/spconv_b200.h.
struct spconv_csr {
    int device = 0;
    bool is_conv = false;
    spb::Geom g{};
    int64_t rows = 0, cols = 0, nnz = 0;
    int k2max = 0;                 // max entries in any row
    bool taps_dense = false;       // every tap non-zero and finite (banded SpMM applies)
    int32_t* row_ptr = nullptr;    // device
    int32_t* col_idx = nullptr;    // device
    float* vals = nullptr;         // device
    float* taps = nullptr;         // device k*k taps (conv transforms)
    uint8_t* seg_ok = nullptr;     // device band-check bytes [mo][tiles_y] (band geometries)
    int band_tw = 0;               // tile width seg_ok was sized for (0: none)
    int64_t sy = 0;                // sum over output columns of the valid tap-column count
    // Storage layout (inc/sparse.hpp:24).  A CSC handle keeps its column-major
    // storage (what export / text / device_ptrs show) next to the row-major
    // arrays above, which every SpMV / SpMM kernel reads.
    // A conv transform built in CSC (build_transform(layout = 1), relayout)
    // keeps ONLY the column-major storage: row_ptr / col_idx / vals are NULL
    // and every apply reads the CSC arrays (csc_apply.cu, conv_band_check<csc>).
    // Matrices that arrive from the host in CSC keep both.
    int layout = 0;                // 0 = CSR, 1 = CSC
    int32_t* csc_ptr = nullptr;    // device col_ptr[cols+1] (layout 1)
    int32_t* csc_idx = nullptr;    // device row_idx[nnz]
    float* csc_vals = nullptr;     // device vals[nnz]
    std::vector<float> host_taps;  // conv handles: the k*k fp32 taps (relayout rebuilds from them)
    // Exact fp64 values, kept only when some value is not an fp32 number
    // (double taps / host values fp32 does not represent): what export, text
    // and the fp64 SpMM read.  The fp32 kernels read vals (narrowed).
    std::vector<double> host_taps64;  // conv handles built from such double taps
    double* vals64 = nullptr;         // device [nnz], row-major order
    double* csc_vals64 = nullptr;     // device [nnz], CSC storage order (layout 1)
    double* taps64 = nullptr;         // device k*k exact taps (CSC conv handles built from double taps)
    int csc_tiles_b = 0;           // CSC band check: segments per input row (band geometries)
    int* fail_flag = nullptr;      // CSC conv: mapped host word, set by a device check that failed (sticky)
    std::atomic<bool> exposed{false};
    std::atomic<bool> checked{false};  // a band check has been enqueued (seg_ok holds verdicts)  // spconv_csr_device_ptrs handed out the CSC arrays: verify before use
    cudaEvent_t built = nullptr;  // recorded after the build on the build stream (host-buffer calls wait on it)
    std::atomic<bool> build_seen{false};  // the built event has been observed complete
    std::atomic<bool> applied{false};  // an apply was enqueued after the build (PDL is safe from then on)
    std::atomic<const char*> last_kernel{nullptr};  // diagnostics: last SpMM kernel launched
    // Workspace of spconv_convolve_host (lazily created, guarded by ws_mu).
    std::mutex ws_mu;
    cudaStream_t ws_stream[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t ws_ev[3][2] = {};
    float* ws_x[2] = {nullptr, nullptr};
    float* ws_y[2] = {nullptr, nullptr};
    int64_t ws_chunk = 0;
    bool ws_built_waited = false;  // the workspace streams are ordered after the build
};
