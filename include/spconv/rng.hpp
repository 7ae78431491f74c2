// Drop-in replacement for the reference's spconv/rng.hpp (inc/rng.hpp:22-98):
// the seeded input generator the reference's benches and verification sweep
// draw from, served by libspconv_b200 (spconv_derive_seed /
// spconv_random_normal) so a reference user's seeds give the same numbers.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "spconv/conv.hpp"
#include "spconv/grid.hpp"
#include "spconv_b200.h"

namespace spconv {

/// Per-index stream seed derived from a base seed.
inline std::uint64_t derive_seed(std::uint64_t base, std::uint64_t index) {
    return spconv_derive_seed(base, index);
}

/// rows x cols standard-normal grid of the stream `seed`.
inline Grid random_normal_grid(index_t rows, index_t cols, std::uint64_t seed) {
    Grid g(rows, cols);
    detail::check(spconv_random_normal(seed, rows * cols, g.values.data()));
    return g;
}

/// k x k standard-normal kernel of the stream `seed`.
inline Kernel random_normal_kernel(index_t k, std::uint64_t seed) {
    std::vector<double> v(static_cast<std::size_t>(k * k));
    detail::check(spconv_random_normal(seed, k * k, v.data()));
    return Kernel(k, std::move(v));
}

}  // namespace spconv
