// Drop-in replacement for the reference's spconv/conv.hpp hot path
// (inc/conv.hpp:33-96 ConvSpec/Kernel, :165-215 Transform/build_transform/
// convolve).  build_transform builds T = C*P directly on the GPU through the
// C ABI (include/spconv_b200.h); convolve / convolve_batch apply it there.
// Both TransformRoute values produce the same matrix, as in the reference.
#pragma once

#include <cstdint>
#include <istream>
#include <iterator>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "spconv/grid.hpp"
#include "spconv/sparse.hpp"
#include "spconv_b200.h"

namespace spconv {

/// m x n input, k x k kernel, stride s, symmetric zero padding p.
struct ConvSpec {
    index_t m = 1, n = 1, k = 1, s = 1, p = 0;

    ConvSpec(index_t m_, index_t n_, index_t k_, index_t s_, index_t p_)
        : m(m_), n(n_), k(k_), s(s_), p(p_) {
        detail::check(spconv_spec_check(m, n, k, s, p));  // same two messages
    }

    index_t padded_rows() const { return m + 2 * p; }
    index_t padded_cols() const { return n + 2 * p; }
    index_t m_out() const { return (padded_rows() - k) / s + 1; }
    index_t n_out() const { return (padded_cols() - k) / s + 1; }
    index_t col_remainder() const { return padded_cols() - k - s * (n_out() - 1); }
    index_t row_remainder() const { return padded_rows() - k - s * (m_out() - 1); }
    index_t vertical_slides() const { return m_out() - 1; }
    index_t input_len() const { return m * n; }
    index_t padded_len() const { return padded_rows() * padded_cols(); }
    index_t output_len() const { return m_out() * n_out(); }

    std::string str() const {
        std::ostringstream os;
        os << "(m=" << m << ", n=" << n << ", k=" << k << ", s=" << s << ", p=" << p << ")";
        return os.str();
    }

    bool operator==(const ConvSpec&) const = default;
};

/// Dense k x k kernel, row-major, placed unflipped (correlation).
struct Kernel {
    index_t k = 1;
    std::vector<double> values;

    Kernel(index_t k_, std::vector<double> v) : k(k_), values(std::move(v)) {
        if (k < 1) throw std::invalid_argument("Kernel: side must be >= 1");
        if (static_cast<index_t>(values.size()) != k * k)
            throw std::invalid_argument("Kernel: expected " + std::to_string(k * k) +
                                        " values, got " + std::to_string(values.size()));
    }

    explicit Kernel(const Grid& g) : Kernel(g.rows, g.values) {
        if (g.rows != g.cols)
            throw std::invalid_argument("Kernel: grid is " + std::to_string(g.rows) + "x" +
                                        std::to_string(g.cols) + ", expected square");
    }

    double at(index_t j, index_t i) const { return values[static_cast<std::size_t>(j * k + i)]; }
};

/// The kernel rotated by 180 degrees (inc/conv.hpp:98-109): passing
/// flipped(K) gives textbook convolution instead of correlation.
inline Kernel flipped(const Kernel& kern) {
    std::vector<double> v(kern.values.rbegin(), kern.values.rend());  // (j, i) -> (k-1-j, k-1-i)
    return Kernel(kern.k, std::move(v));
}

inline DenseVector vectorize(const Grid& a) { return a.values; }

inline Grid unvectorize(DenseVector x, index_t rows, index_t cols) {
    if (static_cast<index_t>(x.size()) != rows * cols)
        throw std::invalid_argument("unvectorize: vector length " + std::to_string(x.size()) +
                                    " does not match " + std::to_string(rows) + "x" +
                                    std::to_string(cols));
    return Grid(rows, cols, std::move(x));
}

/// The composed operator T = C*P (device-resident) with its geometry.
struct Transform {
    ConvSpec spec;
    SparseMatrix matrix;
};

enum class TransformRoute { Spgemm, ColumnGather };

/// P (inc/conv.hpp:125-135): the padding selector, built on the device.
inline SparseMatrix build_padding_matrix(const ConvSpec& spec, Layout layout = Layout::CSR) {
    spconv_csr* h = nullptr;
    detail::check(spconv_build_padding_matrix(spec.m, spec.n, spec.k, spec.s, spec.p, layout == Layout::CSR ? 0 : 1,
                                              detail::default_device(), nullptr, &h));
    return SparseMatrix(h);
}

/// C (inc/conv.hpp:141-162): every tap of every placement, zeros included,
/// built on the device.  build_transform == spgemm(C, P) (its Spgemm route).
inline SparseMatrix build_conv_matrix(const Kernel& kern, const ConvSpec& spec, Layout layout = Layout::CSR) {
    if (kern.k != spec.k)
        throw std::invalid_argument("build_conv_matrix: kernel side " + std::to_string(kern.k) +
                                    " does not match spec " + spec.str());
    spconv_csr* h = nullptr;
    detail::check(spconv_build_conv_matrix(spec.m, spec.n, spec.k, spec.s, spec.p, kern.values.data(),
                                           layout == Layout::CSR ? 0 : 1, detail::default_device(), nullptr, &h));
    return SparseMatrix(h);
}

/// One-time on-device build of T (replaces inc/conv.hpp:179-204).  Entries
/// are stored where the double tap is non-zero, with their exact double
/// values (ptr/idx/val, write_transform and convolve match the reference bit
/// for bit); the fp32 batch kernels apply the taps narrowed to fp32.
inline Transform build_transform(const Kernel& kern, const ConvSpec& spec,
                                 Layout layout = Layout::CSR,
                                 TransformRoute route = TransformRoute::Spgemm) {
    (void)route;  // both reference routes yield the identical matrix
    if (kern.k != spec.k)
        throw std::invalid_argument("build_conv_matrix: kernel side " + std::to_string(kern.k) +
                                    " does not match spec " + spec.str());
    spconv_csr* h = nullptr;
    detail::check(spconv_build_transform_f64(spec.m, spec.n, spec.k, spec.s, spec.p, kern.values.data(),
                                             layout == Layout::CSR ? 0 : 1, detail::default_device(),
                                             nullptr, &h));
    return Transform{spec, SparseMatrix(h)};
}

/// vec, SpMV, reshape (inc/conv.hpp:207-215) on the GPU.
inline Grid convolve(const Transform& t, const Grid& a, int threads = 0) {
    const int nt = threads > 0 ? threads : thread_cap();
    if (a.rows != t.spec.m || a.cols != t.spec.n)
        throw std::invalid_argument("convolve: input is " + std::to_string(a.rows) + "x" +
                                    std::to_string(a.cols) + " but transform expects " +
                                    t.spec.str());
    DenseVector out(static_cast<std::size_t>(t.spec.output_len()));
    detail::check(spconv_convolve_host_f64_threads(t.matrix.handle(), a.values.data(), out.data(), 1, nt));
    return Grid(t.spec.m_out(), t.spec.n_out(), std::move(out));
}

/// Grouped apply (new): each transform applied to its own image in one device
/// call -- a network's layer loop (the reference calls convolve per layer,
/// inc/bench.hpp:240-248).  fp64 in the reference's arithmetic: every output
/// is bit-identical to convolve(*ts[i], images[i]) (threads = 1).
inline std::vector<Grid> convolve_group(const std::vector<const Transform*>& ts, const std::vector<Grid>& images) {
    if (ts.size() != images.size())
        throw std::invalid_argument("convolve_group: " + std::to_string(ts.size()) + " transforms but " +
                                    std::to_string(images.size()) + " images");
    std::vector<const spconv_csr*> hs(ts.size());
    std::vector<const double*> xs(ts.size());
    std::vector<double*> ys(ts.size());
    std::vector<Grid> out;
    out.reserve(ts.size());
    for (std::size_t i = 0; i < ts.size(); ++i) {
        const Transform& t = *ts[i];
        const Grid& a = images[i];
        if (a.rows != t.spec.m || a.cols != t.spec.n)
            throw std::invalid_argument("convolve: input is " + std::to_string(a.rows) + "x" +
                                        std::to_string(a.cols) + " but transform expects " + t.spec.str());
        out.emplace_back(t.spec.m_out(), t.spec.n_out(), DenseVector(static_cast<std::size_t>(t.spec.output_len())));
        hs[i] = t.matrix.handle();
        xs[i] = a.values.data();
        ys[i] = out.back().values.data();
    }
    detail::check(spconv_convolve_host_group_f64(hs.data(), static_cast<int64_t>(ts.size()), xs.data(), ys.data()));
    return out;
}

/// Batch apply (new; the reference loops convolve per image): `images`
/// grids of m x n in, m_out x n_out out, one pipelined device pass.
inline std::vector<Grid> convolve_batch(const Transform& t, const std::vector<Grid>& images) {
    const index_t in = t.spec.input_len(), outl = t.spec.output_len();
    std::vector<float> x(static_cast<std::size_t>(in) * images.size());
    for (std::size_t b = 0; b < images.size(); ++b) {
        const Grid& a = images[b];
        if (a.rows != t.spec.m || a.cols != t.spec.n)
            throw std::invalid_argument("convolve: input is " + std::to_string(a.rows) + "x" +
                                        std::to_string(a.cols) + " but transform expects " +
                                        t.spec.str());
        for (index_t i = 0; i < in; ++i) x[b * in + i] = static_cast<float>(a.values[i]);
    }
    std::vector<float> y(static_cast<std::size_t>(outl) * images.size());
    detail::check(spconv_convolve_host(t.matrix.handle(), x.data(), y.data(),
                                       static_cast<int64_t>(images.size())));
    std::vector<Grid> out;
    out.reserve(images.size());
    for (std::size_t b = 0; b < images.size(); ++b)
        out.emplace_back(t.spec.m_out(), t.spec.n_out(),
                         std::vector<double>(y.begin() + b * outl, y.begin() + (b + 1) * outl));
    return out;
}

/// write_transform (inc/conv.hpp:221-224): the text is rendered on the GPU,
/// byte-identical to the reference's for the same matrix.
inline void write_transform(std::ostream& os, const Transform& t) {
    int64_t len = 0;
    detail::check(spconv_csr_write_text(t.matrix.handle(), 1, nullptr, 0, &len));
    std::string buf(static_cast<std::size_t>(len), '\0');
    detail::check(spconv_csr_write_text(t.matrix.handle(), 1, buf.data(), len, &len));
    os.write(buf.data(), static_cast<std::streamsize>(len));
}

/// read_transform (inc/conv.hpp:226-244); values are kept exactly.
inline Transform read_transform(std::istream& is) {
    std::string text((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
    spconv_csr* h = nullptr;
    detail::check(spconv_transform_read(text.data(), static_cast<int64_t>(text.size()),
                                        detail::default_device(), nullptr, &h));
    SparseMatrix mat(h);
    int64_t s5[5];
    detail::check(spconv_csr_spec(h, s5));
    return Transform{ConvSpec(s5[0], s5[1], s5[2], s5[3], s5[4]), std::move(mat)};
}

}  // namespace spconv
