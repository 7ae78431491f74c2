// Drop-in replacement for the compressed-matrix part of the reference's
// spconv/sparse.hpp (inc/sparse.hpp:24-32, 77-140, 209-274).  A SparseMatrix
// here is a handle on a DEVICE-resident matrix (int32 indices, fp32 values) in
// CSR or CSC layout, built by libspconv_b200; the reference's host accessors
// ptr()/idx()/val() still work and return the storage (in the matrix's
// layout) widened to int64/double, exported lazily on first use.  spmv() runs
// on the GPU (fp32, column-ascending fmaf per output, which is also what the
// reference's one-thread CSC scatter computes) -- there is no CPU path.
#pragma once

#include <cstdlib>
#include <istream>
#include <iterator>
#include <memory>
#include <mutex>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "spconv/grid.hpp"
#include "spconv_b200.h"

namespace spconv {

enum class Layout { CSR, CSC };

inline const char* layout_name(Layout l) { return l == Layout::CSR ? "csr" : "csc"; }

inline Layout layout_from_name(const std::string& s) {
    if (s == "csr" || s == "CSR") return Layout::CSR;
    if (s == "csc" || s == "CSC") return Layout::CSC;
    throw std::invalid_argument("unknown layout '" + s + "' (expected csr or csc)");
}

namespace detail {

/// Maps a C-ABI status to the reference's exception types.
inline void check(int rc) {
    if (rc == SPCONV_OK) return;
    if (rc == SPCONV_EINVAL) throw std::invalid_argument(spconv_last_error());
    throw std::runtime_error(spconv_last_error());
}

struct CsrHandle {
    spconv_csr* h = nullptr;
    explicit CsrHandle(spconv_csr* p) : h(p) {}
    CsrHandle(const CsrHandle&) = delete;
    CsrHandle& operator=(const CsrHandle&) = delete;
    ~CsrHandle() { spconv_csr_free(h); }
};

/// Device ordinal used by the drop-in API (SPCONV_DEVICE, default 0).
inline int default_device() {
    const char* e = std::getenv("SPCONV_DEVICE");
    return e ? std::atoi(e) : 0;
}

}  // namespace detail

/// One stored coordinate (inc/sparse.hpp:35-40).
struct Entry {
    index_t row;
    index_t col;
    double value;
};

/// Coordinate-format builder (inc/sparse.hpp:40-73): same checks and messages.
/// SparseMatrix::compile turns it into compressed storage on the device.
class Triplets {
public:
    Triplets(index_t rows, index_t cols) : rows_(rows), cols_(cols) {
        if (rows < 1 || cols < 1)
            throw std::invalid_argument("Triplets: dimensions must be at least 1x1, got " + std::to_string(rows) +
                                        "x" + std::to_string(cols));
    }

    void reserve(std::size_t n) { entries_.reserve(n); }

    void add(index_t row, index_t col, double value) {
        if (row < 0 || row >= rows_ || col < 0 || col >= cols_)
            throw std::invalid_argument("Triplets: entry (" + std::to_string(row) + ", " + std::to_string(col) +
                                        ") outside " + std::to_string(rows_) + "x" + std::to_string(cols_));
        entries_.push_back({row, col, value});
    }

    index_t rows() const { return rows_; }
    index_t cols() const { return cols_; }
    std::size_t size() const { return entries_.size(); }
    const std::vector<Entry>& entries() const { return entries_; }

private:
    index_t rows_, cols_;
    std::vector<Entry> entries_;
};

/// Compressed sparse matrix resident on the GPU, CSR or CSC.  Copies share the
/// immutable device matrix.
class SparseMatrix {
public:
    SparseMatrix() = default;

    /// Adopts a C-ABI handle (takes ownership).
    explicit SparseMatrix(spconv_csr* h) : dev_(std::make_shared<detail::CsrHandle>(h)) {
        detail::check(spconv_csr_shape(h, &rows_, &cols_, &nnz_));
        int lay = 0;
        detail::check(spconv_csr_layout(h, &lay));
        layout_ = lay == 0 ? Layout::CSR : Layout::CSC;
        host_ = std::make_shared<HostCopy>();
    }

    /// compile (inc/sparse.hpp:85-119): sorted into `layout` order on the device,
    /// duplicates rejected with the reference's message, explicit zeros kept.
    static SparseMatrix compile(const Triplets& t, Layout layout) {
        const std::size_t n = t.size();
        std::vector<index_t> r(n), c(n);
        std::vector<double> v(n);
        for (std::size_t i = 0; i < n; ++i) {
            r[i] = t.entries()[i].row;
            c[i] = t.entries()[i].col;
            v[i] = t.entries()[i].value;
        }
        spconv_csr* h = nullptr;
        detail::check(spconv_matrix_from_coo(t.rows(), t.cols(), static_cast<int64_t>(n), r.data(), c.data(),
                                             v.data(), layout == Layout::CSR ? 0 : 1, detail::default_device(),
                                             nullptr, &h));
        return SparseMatrix(h);
    }

    /// Uploads a host CSR (ptr/idx int64, fp64 values; the fp32 kernels read them narrowed).
    static SparseMatrix from_csr(index_t rows, index_t cols, const std::vector<index_t>& ptr,
                                 const std::vector<index_t>& idx, const std::vector<double>& val) {
        if (static_cast<index_t>(ptr.size()) != rows + 1)
            throw std::invalid_argument("SparseMatrix: ptr must have rows+1 entries");
        spconv_csr* h = nullptr;
        detail::check(spconv_csr_from_host(rows, cols, ptr.data(), idx.data(), val.data(),
                                           detail::default_device(), nullptr, &h));
        return SparseMatrix(h);
    }

    /// Uploads host storage in either layout (ptr over the major dimension).
    static SparseMatrix from_storage(Layout layout, index_t rows, index_t cols,
                                     const std::vector<index_t>& ptr, const std::vector<index_t>& idx,
                                     const std::vector<double>& val) {
        const index_t major = layout == Layout::CSR ? rows : cols;
        if (static_cast<index_t>(ptr.size()) != major + 1)
            throw std::invalid_argument("SparseMatrix: ptr must have major_dim+1 entries");
        spconv_csr* h = nullptr;
        detail::check(spconv_matrix_from_host(rows, cols, layout == Layout::CSR ? 0 : 1, ptr.data(),
                                              idx.data(), val.data(), detail::default_device(),
                                              nullptr, &h));
        return SparseMatrix(h);
    }

    Layout layout() const { return layout_; }
    index_t rows() const { return rows_; }
    index_t cols() const { return cols_; }
    index_t nnz() const { return nnz_; }
    index_t major_dim() const { return layout_ == Layout::CSR ? rows_ : cols_; }
    index_t minor_dim() const { return layout_ == Layout::CSR ? cols_ : rows_; }

    const std::vector<index_t>& ptr() const { return exported().ptr; }
    const std::vector<index_t>& idx() const { return exported().idx; }
    const std::vector<double>& val() const { return exported().val; }

    /// Stored entries in storage order (row-major for CSR, column-major for
    /// CSC), from the exported storage (inc/sparse.hpp:133-149).
    std::vector<Entry> entries() const {
        const HostCopy& hc = exported();
        std::vector<Entry> out;
        out.reserve(static_cast<std::size_t>(nnz_));
        const bool csr = layout_ == Layout::CSR;
        for (index_t maj = 0; maj < major_dim(); ++maj)
            for (index_t e = hc.ptr[static_cast<std::size_t>(maj)]; e < hc.ptr[static_cast<std::size_t>(maj) + 1]; ++e) {
                const index_t mn = hc.idx[static_cast<std::size_t>(e)];
                out.push_back(Entry{csr ? maj : mn, csr ? mn : maj, hc.val[static_cast<std::size_t>(e)]});
            }
        return out;
    }

    /// Row-major dense expansion (inc/sparse.hpp:152-158).
    std::vector<double> to_dense() const {
        std::vector<double> d(static_cast<std::size_t>(rows_ * cols_), 0.0);
        for (const Entry& e : entries()) d[static_cast<std::size_t>(e.row * cols_ + e.col)] = e.value;
        return d;
    }

    /// The C-ABI handle (nullptr for a default-constructed matrix).
    spconv_csr* handle() const { return dev_ ? dev_->h : nullptr; }

private:
    struct HostCopy {
        std::once_flag once;
        std::vector<index_t> ptr, idx;
        std::vector<double> val;
    };
    const HostCopy& exported() const {
        if (!dev_) throw std::logic_error("SparseMatrix: empty matrix");
        std::call_once(host_->once, [this] {
            host_->ptr.resize(static_cast<std::size_t>(major_dim()) + 1);
            host_->idx.resize(static_cast<std::size_t>(nnz_));
            host_->val.resize(static_cast<std::size_t>(nnz_));
            detail::check(spconv_csr_export(dev_->h, host_->ptr.data(), host_->idx.data(),
                                            host_->val.data()));
        });
        return *host_;
    }

    std::shared_ptr<detail::CsrHandle> dev_;
    std::shared_ptr<HostCopy> host_;
    Layout layout_ = Layout::CSR;
    index_t rows_ = 0, cols_ = 0, nnz_ = 0;
};

/// relayout (inc/sparse.hpp:268-274): the same matrix in `layout`.
inline SparseMatrix relayout(const SparseMatrix& m, Layout layout) {
    if (m.layout() == layout) return m;
    spconv_csr* h = nullptr;
    detail::check(spconv_relayout(m.handle(), layout == Layout::CSR ? 0 : 1, nullptr, &h));
    return SparseMatrix(h);
}

/// transposed / pruned / hstack_blocks / vstack_blocks (inc/sparse.hpp:276-395):
/// the entries restaged as Triplets and compiled on the device (same checks,
/// messages and results).
inline SparseMatrix transposed(const SparseMatrix& m) {
    Triplets t(m.cols(), m.rows());
    t.reserve(static_cast<std::size_t>(m.nnz()));
    for (const Entry& e : m.entries()) t.add(e.col, e.row, e.value);
    return SparseMatrix::compile(t, m.layout());
}

inline SparseMatrix pruned(const SparseMatrix& m) {
    Triplets t(m.rows(), m.cols());
    t.reserve(static_cast<std::size_t>(m.nnz()));
    for (const Entry& e : m.entries())
        if (e.value != 0.0) t.add(e.row, e.col, e.value);
    return SparseMatrix::compile(t, m.layout());
}

namespace detail {
// hstack (along = true: columns) / vstack: shared checks, offsets, compile.
inline SparseMatrix stack_blocks(std::span<const SparseMatrix> blocks, Layout out_layout, bool along_cols) {
    const char* name = along_cols ? "hstack_blocks" : "vstack_blocks";
    if (blocks.empty()) throw std::invalid_argument(std::string(name) + ": no blocks");
    const index_t shared = along_cols ? blocks[0].rows() : blocks[0].cols();
    index_t extent = 0;
    std::size_t nnz = 0;
    for (std::size_t b = 0; b < blocks.size(); ++b) {
        const index_t have = along_cols ? blocks[b].rows() : blocks[b].cols();
        if (have != shared)
            throw std::invalid_argument(std::string(name) + ": block " + std::to_string(b) + " has " +
                                        std::to_string(have) + (along_cols ? " rows" : " cols") + ", expected " +
                                        std::to_string(shared));
        extent += along_cols ? blocks[b].cols() : blocks[b].rows();
        nnz += static_cast<std::size_t>(blocks[b].nnz());
    }
    Triplets t(along_cols ? shared : extent, along_cols ? extent : shared);
    t.reserve(nnz);
    index_t off = 0;
    for (const SparseMatrix& blk : blocks) {
        for (const Entry& e : blk.entries())
            t.add(along_cols ? e.row : off + e.row, along_cols ? off + e.col : e.col, e.value);
        off += along_cols ? blk.cols() : blk.rows();
    }
    return SparseMatrix::compile(t, out_layout);
}
}  // namespace detail

inline SparseMatrix hstack_blocks(std::span<const SparseMatrix> blocks, Layout out_layout = Layout::CSR) {
    return detail::stack_blocks(blocks, out_layout, true);
}

inline SparseMatrix vstack_blocks(std::span<const SparseMatrix> blocks, Layout out_layout = Layout::CSR) {
    return detail::stack_blocks(blocks, out_layout, false);
}

/// spgemm (inc/sparse.hpp:296-342), on the device: the reference's Gustavson
/// sums bit for bit in fp64, exact zeros dropped.
inline SparseMatrix spgemm(const SparseMatrix& a, const SparseMatrix& b, Layout out_layout = Layout::CSR) {
    if (a.cols() != b.rows())
        throw std::invalid_argument("spgemm: inner dimensions differ, " + std::to_string(a.cols()) + " vs " +
                                    std::to_string(b.rows()));
    spconv_csr* h = nullptr;
    detail::check(spconv_spgemm(a.handle(), b.handle(), out_layout == Layout::CSR ? 0 : 1, nullptr, &h));
    return SparseMatrix(h);
}

/// Thread count used by spmv when the caller does not pass one
/// (inc/sparse.hpp:171-176): SPCONV_THREADS, default 1.  On the device it
/// selects only the reference's CSC partial-combine order (results of the
/// reference's CSR path do not depend on it).
inline int thread_cap() {
    const char* env = std::getenv("SPCONV_THREADS");
    if (env == nullptr) return 1;
    const long v = std::strtol(env, nullptr, 10);
    return v >= 1 ? static_cast<int>(v) : 1;
}

/// y = M x (inc/sparse.hpp:214-261) in fp64 on the GPU, bit-identical to the
/// reference's spmv(m, x, threads) -- for CSC storage including its
/// per-thread partial combine (spconv_convolve_host_f64_threads).
inline DenseVector spmv(const SparseMatrix& m, std::span<const double> x, int threads = 0) {
    const int nt = threads > 0 ? threads : thread_cap();
    if (m.cols() != static_cast<index_t>(x.size()))
        throw std::invalid_argument("spmv: matrix has " + std::to_string(m.cols()) +
                                    " columns but vector has " + std::to_string(x.size()) +
                                    " elements");
    DenseVector y(static_cast<std::size_t>(m.rows()), 0.0);
    detail::check(spconv_convolve_host_f64_threads(m.handle(), x.data(), y.data(), 1, nt));
    return y;
}

inline DenseVector spmv(const SparseMatrix& m, const DenseVector& x, int threads = 0) {
    return spmv(m, std::span<const double>(x), threads);
}

/// read_sparse (inc/sparse.hpp:409-432): values kept exactly (fp32 kernels read them narrowed).
inline SparseMatrix read_sparse(std::istream& is, Layout layout = Layout::CSR) {
    std::string text((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
    spconv_csr* h = nullptr;
    detail::check(spconv_sparse_read(text.data(), static_cast<int64_t>(text.size()), layout == Layout::CSR ? 0 : 1,
                                     detail::default_device(), nullptr, &h));
    return SparseMatrix(h);
}

/// write_sparse (inc/sparse.hpp:400-406), rendered on the GPU.
inline void write_sparse(std::ostream& os, const SparseMatrix& m) {
    int64_t len = 0;
    detail::check(spconv_csr_write_text(m.handle(), 0, nullptr, 0, &len));
    std::string buf(static_cast<std::size_t>(len), '\0');
    detail::check(spconv_csr_write_text(m.handle(), 0, buf.data(), len, &len));
    os.write(buf.data(), static_cast<std::streamsize>(len));
}

}  // namespace spconv
