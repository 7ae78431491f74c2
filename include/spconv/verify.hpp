// Drop-in replacement for the reference's spconv/verify.hpp
// (inc/verify.hpp:24-169): the exhaustive small-size sweep, run against the
// DEVICE path -- the CSR transform (built from the double taps, exact values)
// and its CSC relayout built and applied on the GPU.  The reference's own
// check runs in fp64 on the device (fp64 SpMM of both layouts vs the fp64
// direct_conv / im2col comparators, bit-identical to inc/reference.hpp), so
// max_conv_dev / max_layout_dev are the reference's numbers.  The fp32 batch
// path is checked on the same handles: bit-equal to the fp32 direct_conv,
// CSR == CSC, and within 1e-5 * sum|w*a| of fp64 (max_rel_dev, an extra field).
#pragma once

#include <cstdint>
#include <sstream>
#include <string>
#include <vector>

#include "spconv/sparse.hpp"
#include "spconv_b200.h"

namespace spconv {

struct VerifyOptions {
    index_t max_dim = 12;
    int seeds = 3;
    std::uint64_t base_seed = 42;
    double conv_tol = 1e-10;    ///< fp64 comparators against each other (fixed in the library)
    double layout_tol = 1e-12;  ///< CSR vs CSC (the device path requires bit equality)
    std::size_t max_failures = 20;
};

struct VerifyReport {
    index_t specs = 0;
    index_t conv_cases = 0;
    index_t clipped_specs = 0;
    double max_conv_dev = 0.0;
    double max_layout_dev = 0.0;
    double max_rel_dev = 0.0;  ///< max |y_fp32 - y_ref| / sum|w*a| (device path)
    std::vector<std::string> failures;

    bool ok() const { return failures.empty(); }
};

inline VerifyReport run_verification(const VerifyOptions& opt = {}) {
    std::int64_t counts[4] = {0, 0, 0, 0};
    double devs[3] = {0, 0, 0};
    std::string buf(16384, '\0');
    detail::check(spconv_run_verification(opt.max_dim, opt.seeds, opt.base_seed, detail::default_device(),
                                          counts, devs, buf.data(), static_cast<std::int64_t>(buf.size())));
    VerifyReport rep;
    rep.specs = counts[0];
    rep.conv_cases = counts[1];
    rep.clipped_specs = counts[2];
    rep.max_conv_dev = devs[0];
    rep.max_layout_dev = devs[1];
    rep.max_rel_dev = devs[2];
    std::istringstream is(buf.c_str());
    for (std::string line; std::getline(is, line);)
        if (!line.empty() && rep.failures.size() < opt.max_failures) rep.failures.push_back(line);
    return rep;
}

}  // namespace spconv
