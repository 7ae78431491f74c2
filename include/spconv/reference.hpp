// Drop-in replacement for the reference's spconv/reference.hpp
// (inc/reference.hpp:41-136): the dense comparators -- direct sliding window,
// im2col lowering, im2col product -- with the reference's signatures and
// messages, computed on the GPU in fp64 with the reference's own arithmetic
// (one rounded multiply and one rounded add per tap, (j, i) order, padding
// taps included), so the results are bit-identical to the reference's.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "spconv/conv.hpp"
#include "spconv/grid.hpp"
#include "spconv_b200.h"

namespace spconv {

namespace detail {

inline void check_input_dims(const Grid& a, const ConvSpec& spec, const char* who) {
    if (a.rows != spec.m || a.cols != spec.n)
        throw std::invalid_argument(std::string(who) + ": input is " + std::to_string(a.rows) + "x" +
                                    std::to_string(a.cols) + " but spec is " + spec.str());
}

inline void check_kernel_side(const Kernel& kern, const ConvSpec& spec, const char* who) {
    if (kern.k != spec.k)
        throw std::invalid_argument(std::string(who) + ": kernel side " + std::to_string(kern.k) +
                                    " does not match spec " + spec.str());
}

}  // namespace detail

/// out[x][y] = sum_{j,i} K[j][i] * Apad[s*x+j][s*y+i] (inc/reference.hpp:41-61).
inline Grid direct_conv(const Grid& a, const Kernel& kern, const ConvSpec& spec) {
    detail::check_input_dims(a, spec, "direct_conv");
    detail::check_kernel_side(kern, spec, "direct_conv");
    Grid out(spec.m_out(), spec.n_out());
    detail::check(spconv_reference_host(0, spec.m, spec.n, spec.k, spec.s, spec.p, kern.values.data(),
                                        a.values.data(), out.values.data(), detail::default_device()));
    return out;
}

/// Dense k^2 x (m_out*n_out) patch matrix, row-major (inc/reference.hpp:63-71).
struct Im2colMatrix {
    index_t rows = 0;
    index_t cols = 0;
    std::vector<double> values;
};

/// The explicit lowering (inc/reference.hpp:73-97), built on the GPU.
inline Im2colMatrix im2col(const Grid& a, const ConvSpec& spec) {
    detail::check_input_dims(a, spec, "im2col");
    const index_t k2 = spec.k * spec.k, patches = spec.output_len();
    Im2colMatrix m{k2, patches, std::vector<double>(static_cast<std::size_t>(k2 * patches))};
    detail::check(spconv_reference_host(2, spec.m, spec.n, spec.k, spec.s, spec.p, nullptr, a.values.data(),
                                        m.values.data(), detail::default_device()));
    return m;
}

/// im2col lowering plus dense product (inc/reference.hpp:120-127).
inline Grid im2col_conv(const Grid& a, const Kernel& kern, const ConvSpec& spec) {
    detail::check_kernel_side(kern, spec, "im2col_conv");
    detail::check_input_dims(a, spec, "im2col");
    Grid out(spec.m_out(), spec.n_out());
    detail::check(spconv_reference_host(1, spec.m, spec.n, spec.k, spec.s, spec.p, kern.values.data(),
                                        a.values.data(), out.values.data(), detail::default_device()));
    return out;
}

}  // namespace spconv
