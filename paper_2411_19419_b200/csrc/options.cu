// options.cu -- process-wide kernel-path options (spconv_set_option).
//
// The library picks its kernels itself (capi.cu run_spmm, csr_build.cu
// launch_csr_build); these options only force an alternative path, so the
// tests can cross-check every kernel against the oracle and the A/B scripts
// can time the rejected variants.  They are plain atomics read once per call:
// no environment lookups on the call path.
#include <cstring>
#include <string>

#include "../../include/spconv_b200.h"
#include "internal.h"

namespace spb {

std::atomic<int> g_opt[kOptCount] = {};

namespace {

struct OptSpec {
    const char* name;
    Opt id;
    const char* values[8];  // symbolic values, index = stored value; nullptr-terminated (empty: integer)
};

const OptSpec kSpecs[] = {
    {"path", kOptPath, {"auto", "banded", "tiled", "tiled_notma", "generic", "spmv", "spmv_plain", nullptr}},
    {"fused", kOptFused, {"auto", "0", "1", nullptr}},
    {"generic", kOptGeneric, {"rowblock", "plain", nullptr}},
    {"build", kOptBuild, {"auto", "block", "warp", "persist", nullptr}},
    {"bulk_store", kOptBulkStoreOff, {"1", "0", nullptr}},
    {"stage", kOptStage, {"auto", "bulk", "window", nullptr}},
    {"spec_skew", kOptSpecSkew, {nullptr}},
    {"repitch", kOptRepitch, {"auto", "off", nullptr}},
    {"pdl", kOptPdl, {"auto", "off", "apply_only", nullptr}},
};

}  // namespace
}  // namespace spb

extern "C" {

int spconv_set_option(const char* name, const char* value) {
    if (!name || !value) return spb_fail(SPCONV_EINVAL, "spconv_set_option: null argument");
    for (const auto& s : spb::kSpecs) {
        if (std::strcmp(s.name, name)) continue;
        if (!s.values[0]) {  // integer option
            char* end = nullptr;
            const long v = std::strtol(value, &end, 10);
            if (!*value || *end) return spb_fail(SPCONV_EINVAL, std::string("spconv_set_option: ") + name + " takes an integer");
            spb::g_opt[s.id].store((int)v);
            return SPCONV_OK;
        }
        for (int i = 0; s.values[i]; ++i)
            if (!std::strcmp(s.values[i], value)) {
                spb::g_opt[s.id].store(i);
                return SPCONV_OK;
            }
        return spb_fail(SPCONV_EINVAL, std::string("spconv_set_option: bad value '") + value + "' for " + name);
    }
    return spb_fail(SPCONV_EINVAL, std::string("spconv_set_option: unknown option '") + name + "'");
}

int spconv_get_option(const char* name, char* buf, int64_t cap) {
    if (!name || !buf || cap < 1) return spb_fail(SPCONV_EINVAL, "spconv_get_option: null argument");
    for (const auto& s : spb::kSpecs) {
        if (std::strcmp(s.name, name)) continue;
        const int v = spb::g_opt[s.id].load();
        const std::string out = s.values[0] ? std::string(s.values[v]) : std::to_string(v);
        if ((int64_t)out.size() + 1 > cap) return spb_fail(SPCONV_EINVAL, "spconv_get_option: buffer too small");
        std::memcpy(buf, out.c_str(), out.size() + 1);
        return SPCONV_OK;
    }
    return spb_fail(SPCONV_EINVAL, std::string("spconv_get_option: unknown option '") + name + "'");
}

}  // extern "C"
