/*
 * spconv_b200.h -- the C-ABI drop-in boundary of the B200 conv-as-SpMV path.
 *
 * The reference (arxiv 2411.19419 spec implementation, /root/reference/proj)
 * is a header-only C++20 library with no FFI; its "operator API" is the set of
 * inline functions in namespace spconv.  Each entry point below replaces one
 * of them (cited as inc/<file>:<line>, inc = proj/include/spconv) and is what
 * the drop-in C++ headers in include/spconv/ call.  Plain pointers and sizes
 * only; no torch or CUDA types cross this boundary (streams are passed as
 * void* holding a cudaStream_t; NULL = the legacy default stream).
 *
 * Device format of a transform T (m_out*n_out x m*n):
 *   row_ptr int32[rows+1], col_idx int32[nnz], vals float32[nnz]
 * identical in structure to the reference CSR (inc/sparse.hpp:85-119);
 * export widens to the reference's int64/int64/double.
 *
 * Status codes: 0 ok, 1 invalid argument (the reference would throw
 * std::invalid_argument; the message is the reference's), 2 CUDA / out of
 * memory / internal error.  spconv_last_error() returns the calling thread's
 * last message.  A built handle is immutable: concurrent spconv_spmv /
 * spconv_spmm calls on different streams are safe.
 *
 * Stream ordering: a build returns once its kernels are enqueued on `stream`.
 * Device-pointer applies (spconv_spmv / spconv_spmm) on that same stream are
 * ordered after it; on another stream the caller orders them (an event), as
 * with any CUDA producer.  The host-buffer calls (spconv_convolve_host*) and
 * every synchronous call (export, copy, text) wait for the build themselves.
 * From a handle's second apply on, applies are launched as programmatic
 * dependents of the kernel before them on the stream: they may start reading
 * the handle's own storage before that kernel ends, but read x and write y
 * only after it (stream order for the caller's data is unchanged).  Storage
 * handed out by spconv_csr_device_ptrs is never read early (option pdl = off
 * disables the early start altogether).
 */
#ifndef SPCONV_B200_H
#define SPCONV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPCONV_OK 0
#define SPCONV_EINVAL 1
#define SPCONV_ECUDA 2
#define SPCONV_ERUNTIME 3 /* the reference would throw std::runtime_error (I/O, format) */

/* Opaque device-resident CSR (replaces spconv::Transform / SparseMatrix,
 * inc/conv.hpp:165-168, inc/sparse.hpp:77-140). */
typedef struct spconv_csr spconv_csr;

/* Thread-local message for the last non-zero status. */
const char* spconv_last_error(void);

/* ABI version (major*100 + minor). */
int spconv_abi_version(void);

/* ConvSpec validation, inc/conv.hpp:40-48 (same two messages). */
int spconv_spec_check(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p);

/* Theorem 2.1 closed-form count, replaces nnz_bound inc/analysis.hpp:56-66. */
int spconv_nnz_bound(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int64_t* out);

/* One-time on-device CSR build of T = C*P for a k x k kernel (host fp32,
 * row-major, unflipped = correlation).  Replaces build_transform
 * inc/conv.hpp:179-204 (both routes; exact-zero taps are dropped as at
 * inc/sparse.hpp:335 / inc/conv.hpp:201).  Runs on `device` / `stream`; the
 * call returns once the build is enqueued and the handle is valid (the
 * device arrays are complete when `stream` reaches this point). */
int spconv_build_csr(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p,
                     const float* kernel_kxk, int device, void* stream, spconv_csr** out);

/* build_transform(kernel, spec, layout) (inc/conv.hpp:179-204) with the
 * storage layout of inc/sparse.hpp:24: 0 = CSR (same as spconv_build_csr),
 * 1 = CSC -- column c = a*n + b holds its rows in ascending order, built on
 * the device in closed form (csc_build.cu), bit-identical to the reference's
 * compile(..., Layout::CSC).  A CSC conv handle holds ONLY that storage:
 * spconv_spmm / spconv_spmm_f64 read it (detail::spmv_csc_cols,
 * inc/sparse.hpp:194-205, as a per-output gather at closed-form places,
 * csc_apply.cu; for batches of the band geometries a CSC band check feeding
 * the register-blocked apply, spmm_band.cu), checking it against the taps on
 * every call. */
int spconv_build_transform(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p,
                           const float* kernel_kxk, int layout, int device, void* stream,
                           spconv_csr** out);

/* build_transform(kernel, spec, layout) (inc/conv.hpp:179-204) for the
 * reference's own tap type, double.  Entries are kept exactly where the
 * reference keeps them (double tap != 0.0, inc/sparse.hpp:335).  When every
 * tap is an fp32 number this IS spconv_build_transform.  Otherwise the handle
 * also keeps the exact fp64 value of every entry (built on the device from
 * the taps): export, the text writer and spconv_spmm_f64 /
 * spconv_convolve_host_f64 use them -- bit-identical to the reference for any
 * double taps -- while the fp32 kernels (spmv / spmm / convolve_host) apply
 * the fp32-narrowed taps. */
int spconv_build_transform_f64(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p,
                               const double* kernel_kxk, int layout, int device, void* stream,
                               spconv_csr** out);

/* "%.17g" of v as the device text writer renders it (exact: glibc's
 * correctly rounded output), NUL-terminated into out (>= 32 bytes); returns
 * the length.  Host-callable (no device work). */
int spconv_format_g17(double v, char* out);

/* SparseMatrix::layout() (inc/sparse.hpp:121): 0 = CSR, 1 = CSC. */
int spconv_csr_layout(const spconv_csr* h, int* layout);

/* relayout(m, layout) (inc/sparse.hpp:268-274): a new handle holding the same
 * matrix in `layout` (a copy when the layouts agree).  Conv handles are
 * rebuilt on the device from their taps; matrices that came from the host are
 * transposed from a host copy. */
int spconv_relayout(const spconv_csr* h, int layout, void* stream, spconv_csr** out);

/* Uploads a host matrix in either layout: layout 0 = spconv_csr_from_host,
 * layout 1 = CSC (ptr over the cols+1 columns, row indices strictly ascending
 * per column). */
int spconv_matrix_from_host(int64_t rows, int64_t cols, int layout, const int64_t* ptr,
                            const int64_t* idx, const double* vals, int device, void* stream,
                            spconv_csr** out);

/* Uploads an arbitrary host CSR (int64 ptr/idx, double values; the fp32
 * kernels read them narrowed, and when some value is not an fp32 number the
 * exact doubles are kept too, for export / text / the fp64 SpMM) -- the device image of a reference SparseMatrix
 * (inc/sparse.hpp:121-130) for spmv on matrices not built here (e.g. read
 * with read_sparse, inc/sparse.hpp:412-432).  Columns must be strictly
 * ascending per row (the CSR contract of inc/sparse.hpp:77-83). */
int spconv_csr_from_host(int64_t rows, int64_t cols, const int64_t* row_ptr,
                         const int64_t* col_idx, const double* vals, int device, void* stream,
                         spconv_csr** out);

/* SparseMatrix::compile(Triplets, layout) (inc/sparse.hpp:35-119): n host
 * coordinate entries (row[i], col[i], vals[i]) in any order -> a matrix in
 * `layout` (0 = CSR, 1 = CSC), compiled ON THE DEVICE (a radix sort of the
 * (major, minor) keys, duplicate detection, ptr from the key boundaries).
 * Same checks and messages: Triplets' dimension and range checks, and
 * "SparseMatrix: duplicate entry at (r, c)" (status 1).  Explicit zeros are
 * kept; values fp32 cannot hold are kept exactly too (see
 * spconv_csr_from_host).  Synchronous. */
int spconv_matrix_from_coo(int64_t rows, int64_t cols, int64_t n, const int64_t* row, const int64_t* col,
                           const double* vals, int layout, int device, void* stream, spconv_csr** out);

/* spgemm(a, b, layout) (inc/sparse.hpp:296-342) on the device: the products
 * a_ik * b_kj expanded in the reference's order (a's row entries ascending,
 * then b's row k ascending), stable-sorted by (i, j), each run summed in that
 * order from 0.0 with one rounded multiply and one rounded add per product
 * (the reference's Gustavson accumulator, bit for bit), entries that sum to
 * exactly 0.0 dropped.  Operands' exact doubles are used when they keep them.
 * "spgemm: inner dimensions differ, X vs Y" (status 1). */
int spconv_spgemm(const spconv_csr* a, const spconv_csr* b, int layout, void* stream, spconv_csr** out);

/* build_padding_matrix(spec, layout) (inc/conv.hpp:125-135): the selector P,
 * (m+2p)(n+2p) x mn, one 1.0 per input pixel; built on the device. */
int spconv_build_padding_matrix(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int layout, int device,
                                void* stream, spconv_csr** out);

/* build_conv_matrix(kernel, spec, layout) (inc/conv.hpp:141-162): C,
 * m_out*n_out x (m+2p)(n+2p), all k*k taps per row (zeros included) at their
 * padded-grid columns; built on the device, exact doubles kept. */
int spconv_build_conv_matrix(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, const double* kernel_kxk,
                             int layout, int device, void* stream, spconv_csr** out);

/* rows(), cols(), nnz(): inc/sparse.hpp:121-126. */
int spconv_csr_shape(const spconv_csr* h, int64_t* rows, int64_t* cols, int64_t* nnz);

/* Geometry {m,n,k,s,p} of a built transform (Transform::spec,
 * inc/conv.hpp:166); returns 1 for an uploaded generic CSR. */
int spconv_csr_spec(const spconv_csr* h, int64_t spec5[5]);

/* Device pointers of the storage arrays (owned by the handle): ptr over the
 * major dimension (rows for CSR, columns for CSC).  Writing through them is
 * allowed; every later apply follows the storage as it then stands (CSR: the
 * band check re-reads it each call; CSC: once its arrays are handed out, each
 * apply first checks them on the device and waits for the verdict, and an
 * altered storage is applied with the reference's scatter semantics). */
int spconv_csr_device_ptrs(const spconv_csr* h, const int32_t** row_ptr, const int32_t** col_idx,
                           const float** vals);

/* Device bytes of the index / value arrays the handle holds (row-major,
 * column-major, exact-fp64 copies): 8*nnz + 4*(major+1) per layout kept
 * (+ 8*nnz per exact-value array).  A CSC conv transform holds one layout. */
int spconv_csr_storage_bytes(const spconv_csr* h, int64_t* bytes);

/* Synchronous export to host, widened to the reference's types: ptr(),
 * idx(), val() of inc/sparse.hpp:128-130, in the handle's layout (ptr has
 * major_dim()+1 entries).  Any pointer may be NULL. */
int spconv_csr_export(const spconv_csr* h, int64_t* row_ptr, int64_t* col_idx, double* vals);

/* Copies the native device storage arrays (int32 ptr / int32 idx / fp32
 * vals, in the handle's layout) into caller buffers, host or device (any pointer may be NULL),
 * ordered on `stream`; returns when the copies are complete. */
int spconv_csr_copy(const spconv_csr* h, int32_t* row_ptr, int32_t* col_idx, float* vals,
                    void* stream);

/* y = T x on device buffers (fp32).  Replaces spmv inc/sparse.hpp:214-261 /
 * convolve inc/conv.hpp:207-215.  Per row: acc = +0.0f; for each stored
 * entry in column-ascending order acc = fmaf(val, x[col], acc). */
int spconv_spmv(const spconv_csr* h, const float* x_dev, float* y_dev, void* stream);

/* Y[b] = T X[b] for b < batch, image-major device buffers:
 * X[b*ldx + col], Y[b*ldy + row].  The multi-vector form the reference
 * lacks (callers loop convolve per image, inc/bench.hpp:240-248). */
int spconv_spmm(const spconv_csr* h, const float* X_dev, int64_t ldx, float* Y_dev, int64_t ldy,
                int64_t batch, void* stream);

/* End-to-end apply on HOST buffers (X[batch][cols] -> Y[batch][rows], fp32):
 * chunked host->device copy, spmm and device->host copy, overlapped on
 * internal streams; returns when Y is complete.  Pinned buffers give full
 * PCIe overlap. */
int spconv_convolve_host(const spconv_csr* h, const float* X_host, float* Y_host, int64_t batch);

/* Grouped apply: y_dev[i] = T_i x_dev[i] for i < count, every member a
 * transform of its own (one vector each), all on one device, in ONE launch
 * for the CSR members (group.cu); CSC members apply as spconv_spmv would.
 * Each y is bit-identical to spconv_spmv(hs[i], x_dev[i], y_dev[i]).  The y
 * ranges may not overlap each other or any x.  The layer-table loop of
 * inc/bench.hpp:202-349 (one convolve per layer) as a single call. */
int spconv_spmv_group(const spconv_csr* const* hs, int64_t count, const float* const* x_dev,
                      float* const* y_dev, void* stream);

/* spconv_spmv_group on HOST vectors (x_host[i]: cols_i floats, y_host[i]:
 * rows_i floats, any host memory): the inputs are packed into a page-locked
 * staging buffer, copied in one transfer, applied in one launch, and the
 * outputs copied back in one transfer; returns when every y is written. */
int spconv_convolve_host_group(const spconv_csr* const* hs, int64_t count, const float* const* x_host,
                               float* const* y_host);

/* The fp64 forms: the reference's own arithmetic per member (one rounded
 * multiply and one rounded add per entry, inc/sparse.hpp:185-191), each y
 * bit-identical to spconv_spmm_f64 on that member -- and so to the
 * reference's spmv() / convolve() -- in one launch for the CSR members. */
int spconv_spmv_group_f64(const spconv_csr* const* hs, int64_t count, const double* const* x_dev,
                          double* const* y_dev, void* stream);
int spconv_convolve_host_group_f64(const spconv_csr* const* hs, int64_t count, const double* const* x_host,
                                   double* const* y_host);

/* fp64 SpMM on device buffers with the reference's own arithmetic: per row
 * acc = 0.0; acc = acc + (double)val * x[col] over the stored entries in
 * order, one rounded multiply and one rounded add each (inc/sparse.hpp:185-191
 * as its Release build evaluates it).  Bit-identical to the reference's
 * spmv() whenever the stored values equal the reference's: always for
 * handles from spconv_build_transform_f64 / host uploads (they keep exact
 * values when fp32 cannot hold them), and for fp32 taps otherwise. */
int spconv_spmm_f64(const spconv_csr* h, const double* X_dev, int64_t ldx, double* Y_dev, int64_t ldy,
                    int64_t batch, void* stream);

/* spconv_spmm_f64 with the reference's thread count (spmv(m, x, threads),
 * inc/sparse.hpp:214-258): for a CSC matrix with nt = min(threads, cols) > 1
 * the columns are cut into chunks of ceil(cols / nt), each chunk summed into a
 * partial from 0.0 and the partials added to y in chunk order -- the
 * reference's CSC combine, bit for bit.  threads <= 1, or a CSR matrix: the
 * single-thread order (the reference's CSR rows do not depend on it). */
int spconv_spmm_f64_threads(const spconv_csr* h, const double* X_dev, int64_t ldx, double* Y_dev, int64_t ldy,
                            int64_t batch, int threads, void* stream);

/* The reference-semantics apply on fp64 HOST buffers (the reference
 * Grid/DenseVector types, inc/grid.hpp:18-24), used by the drop-in
 * convolve()/spmv(): fp64 in, spconv_spmm_f64 on the device, fp64 out. */
int spconv_convolve_host_f64(const spconv_csr* h, const double* X_host, double* Y_host,
                             int64_t batch);

/* spconv_convolve_host_f64 with the reference's thread count (see
 * spconv_spmm_f64_threads); the drop-in spmv / convolve pass
 * threads > 0 ? threads : thread_cap() (SPCONV_THREADS, inc/sparse.hpp:171-176). */
int spconv_convolve_host_f64_threads(const spconv_csr* h, const double* X_host, double* Y_host,
                                     int64_t batch, int threads);

/* Text form of the matrix, rendered on the device: with
 * transform_header_line != 0, write_transform (inc/conv.hpp:217-224):
 * "%%transform m n k s p csr|csc" then write_sparse (inc/sparse.hpp:400-406):
 * "%%sparse coordinate real", "rows cols nnz", one "row col value" line per
 * entry (1-based, storage order -- column-major for CSC, value = "%.17g" of the entry's
 * exact double when the handle keeps one, else of the fp32 value widened).  Byte-identical to the reference's output for the same matrix.
 * buf == NULL: only *len (the text size in bytes) is computed; otherwise the
 * text is copied to buf (cap >= *len bytes, no terminator). */
int spconv_csr_write_text(const spconv_csr* h, int transform_header_line, char* buf, int64_t cap,
                          int64_t* len);

/* read_transform (inc/conv.hpp:226-244) + read_sparse (inc/sparse.hpp:412-432)
 * of `len` bytes of text: same header checks, range / duplicate checks and
 * messages (status 3 where the reference throws std::runtime_error, 1 for
 * std::invalid_argument).  Values are kept exactly (see spconv_csr_from_host).  A matrix that equals
 * the conv transform of its own taps comes back as a built conv handle
 * (band kernels apply); anything else as a generic CSR with the geometry
 * attached.  The file's layout (csr / csc) is the handle's layout. */
int spconv_transform_read(const char* text, int64_t len, int device, void* stream, spconv_csr** out);

/* The reference's seeded generator (inc/rng.hpp:22-98; host code, no GPU):
 * derive_seed, and `count` standard normals of the stream seeded by `seed`
 * (xoshiro256++ seeded by splitmix64, Marsaglia polar method) -- the inputs
 * random_normal_grid / random_normal_kernel produce. */
uint64_t spconv_derive_seed(uint64_t base, uint64_t index);
int spconv_random_normal(uint64_t seed, int64_t count, double* out);

/* Dense comparators of inc/reference.hpp on the device, over `batch` images
 * (A[b][m*n] -> out[b][m_out*n_out], device buffers, `taps_dev` = k*k taps of
 * the same type).  dtype 1 = fp64 with one rounded multiply and one rounded
 * add per tap in (j, i) order, padding taps included: bit-identical to the
 * reference's direct_conv (inc/reference.hpp:41-61) and im2col_conv
 * (:73-136).  dtype 0 = fp32 fmaf in the same order: the device SpMV's
 * contract (equal to spconv_spmv bit for bit on finite inputs).
 * direct_conv optionally writes sum|w*a| per output to mag_dev (tolerances);
 * im2col_conv materialises the k^2 x (m_out*n_out) patch matrix per image in
 * patches_dev (batch * k^2 * m_out * n_out elements). */
int spconv_direct_conv(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int dtype, const void* taps_dev,
                       const void* A_dev, void* out_dev, void* mag_dev, int64_t batch, void* stream);
int spconv_im2col_conv(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int dtype, const void* taps_dev,
                       const void* A_dev, void* out_dev, void* patches_dev, int64_t batch, void* stream);

/* The same fp64 comparators on HOST buffers for one image (the reference's
 * own signatures, inc/reference.hpp:41-136): mode 0 = direct_conv,
 * 1 = im2col_conv (out: m_out*n_out values), 2 = im2col lowering only (out:
 * the k^2 x m_out*n_out patch matrix, row-major; `kernel` unused).  Computed
 * on `device`, bit-identical to the reference's fp64 results. */
int spconv_reference_host(int mode, int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, const double* kernel,
                          const double* A, double* out, int device);

/* Device-resident timing for the layer-table bench (inc/bench.hpp:202-261 with
 * a GPU method column): `reps` back-to-back applies captured in one CUDA graph,
 * replayed `warmup` times untimed and `trials` times between CUDA events;
 * *mean_us / *sem_us per apply.  method 0 = spconv_spmm of `h` over `batch`
 * device-resident images; method 1 = the fp32 device im2col_conv of
 * (m,n,k,s,p) with `taps_host` (one image; h unused). */
int spconv_time_apply(int method, const spconv_csr* h, int64_t batch, int64_t m, int64_t n, int64_t k, int64_t s,
                      int64_t p, const float* taps_host, int64_t reps, int64_t trials, int64_t warmup,
                      double* mean_us, double* sem_us);

/* run_verification (inc/verify.hpp:59-169) over the device path: for every
 * m, n <= max_dim, p <= 3, s <= 3, k <= min(m,n) + 2p, the Theorem 2.1 count
 * against the brute-force overlap count and nnz(T), and for `seeds` seeded
 * cases (the reference's inputs: derive_seed(base_seed, case), nonzero
 * kernels) the device CSR transform built from the double taps
 * (spconv_build_transform_f64) and its device CSC relayout.  The reference's
 * own check (inc/verify.hpp:124-155), in fp64 on the device: both layouts
 * through spconv_spmm_f64, the fp64 direct_conv and im2col_conv, all within
 * 1e-10 (the reference's conv_tol) and CSR == CSC.  The fp32 contract on the
 * same handles: spmv within 1e-5 * sum|w*a| of the fp64 result on the same
 * fp32-rounded data, BIT-equal to the fp32 direct_conv, CSR == CSC bit for
 * bit.  counts = {specs, conv_cases, clipped_specs, failures}; devs = {the
 * reference's max_conv_dev, max_layout_dev (fp64 leg), max condition-relative
 * fp32 deviation}; `failures` gets the
 * first (at most 20) failure lines, '
'-separated. */
int spconv_run_verification(int64_t max_dim, int seeds, uint64_t base_seed, int device, int64_t counts[4],
                            double devs[3], char* failures, int64_t cap);

/* read_sparse(is, layout) (inc/sparse.hpp:409-432): the coordinate text alone
 * (no transform header) into a generic matrix in `layout` (0 csr, 1 csc);
 * same checks and messages as spconv_transform_read. */
int spconv_sparse_read(const char* text, int64_t len, int layout, int device, void* stream, spconv_csr** out);

/* Name of the kernel(s) the last spconv_spmv / spconv_spmm /
 * spconv_convolve_host call on this handle launched (diagnostics; "" before
 * the first call).  The string is static. */
const char* spconv_csr_last_kernel(const spconv_csr* h);

/* Diagnostics: the verdicts of the last band check run on this handle (one per
 * segment of output columns): *segments = how many, *failed = how many did
 * not match the conv pattern (their rows were computed per entry).  0 failed
 * means the blocked path served every row.  Synchronizes the device; status 1
 * for a handle without band geometry. */
int spconv_band_check_status(const spconv_csr* h, int64_t* segments, int64_t* failed);

/* The per-segment verdicts themselves (1 = the segment's stored entries are
 * the transform's), in segment order: output row x, then column segment
 * (CSR), or input row, then column segment (CSC); *n = the segment count. */
int spconv_band_check_flags(const spconv_csr* h, uint8_t* out, int64_t cap, int64_t* n);

/* Frees the handle and its device memory (synchronises its device). */
int spconv_csr_free(spconv_csr* h);

/* Process-wide kernel-path options (no reference counterpart: the reference
 * has one CPU loop).  The library chooses its kernels itself; an option only
 * forces an alternative so tests can cross-check every kernel and A/B scripts
 * can time the rejected variants.  name = value:
 *   path       auto | banded | tiled | tiled_notma | generic | spmv | spmv_plain
 *   fused      auto | 0 | 1          (band path: two kernels / fused check + apply)
 *   generic    rowblock | plain      (generic CSR batches)
 *   build      auto | block | warp | persist
 *   bulk_store 1 | 0                 (TMA bulk write-back of staged build entries)
 *   stage      lanes | bulk          (latency SpMV staging)
 *   spec_skew  <int>                 (test hook: mispredicts closed-form row starts)
 * Status 1 for an unknown name or value.  spconv_get_option writes the current
 * value (NUL-terminated) into buf. */
int spconv_set_option(const char* name, const char* value);
int spconv_get_option(const char* name, char* buf, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* SPCONV_B200_H */
