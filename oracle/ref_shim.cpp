// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper that compiles the UNMODIFIED reference headers
// (/root/reference/proj/include/spconv/*.hpp, included by path, never copied)
// into oracle/_ref/libspconv_ref.so so that Python tests and the bench's
// reference arm can call the reference's own build_transform / convolve /
// run_verification.  Flags follow the reference Release build
// (proj/CMakeLists.txt:8-10: -O3 -DNDEBUG, gnu++20).  See oracle/Makefile.
//
// Every entry returns 0 on success; on exception it returns 1
// (std::invalid_argument) or 2 (anything else) and stores e.what() for
// ref_last_error().

#include <cstdint>
#include <cstring>
#include <sstream>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "spconv/spconv.hpp"

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_derive_seed(uint64_t base, uint64_t index) { return spconv::derive_seed(base, index); }

int ref_random_normal_grid(int64_t rows, int64_t cols, uint64_t seed, double* out) {
    return guarded([&] {
        const spconv::Grid g = spconv::random_normal_grid(rows, cols, seed);
        std::memcpy(out, g.values.data(), g.values.size() * sizeof(double));
    });
}

int ref_random_normal_kernel(int64_t k, uint64_t seed, double* out) {
    return guarded([&] {
        const spconv::Kernel kern = spconv::random_normal_kernel(k, seed);
        std::memcpy(out, kern.values.data(), kern.values.size() * sizeof(double));
    });
}

int ref_spec_check(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p) {
    return guarded([&] { (void)spconv::ConvSpec(m, n, k, s, p); });
}

int ref_nnz_bound(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int64_t* out) {
    return guarded([&] { *out = spconv::nnz_bound(spconv::ConvSpec(m, n, k, s, p)); });
}

int ref_nnz_oracle(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int64_t* out) {
    return guarded([&] { *out = spconv::nnz_oracle(spconv::ConvSpec(m, n, k, s, p)); });
}

int ref_nnz_per_output(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, int64_t* out) {
    return guarded([&] {
        const auto v = spconv::nnz_per_output(spconv::ConvSpec(m, n, k, s, p));
        std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
    });
}

// Builds T with the reference's build_transform; route 0 = Spgemm (default),
// 1 = ColumnGather.  Returns an owning handle.
int ref_build_transform(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, const double* kern,
                        int route, void** out) {
    return guarded([&] {
        const spconv::ConvSpec spec(m, n, k, s, p);
        const spconv::Kernel kernel(k, std::vector<double>(kern, kern + k * k));
        auto* t = new spconv::Transform(spconv::build_transform(
            kernel, spec, spconv::Layout::CSR,
            route == 0 ? spconv::TransformRoute::Spgemm : spconv::TransformRoute::ColumnGather));
        *out = t;
    });
}

// build_transform with an explicit layout (0 = CSR, 1 = CSC).
int ref_build_transform_layout(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p,
                               const double* kern, int route, int layout, void** out) {
    return guarded([&] {
        const spconv::ConvSpec spec(m, n, k, s, p);
        const spconv::Kernel kernel(k, std::vector<double>(kern, kern + k * k));
        auto* t = new spconv::Transform(spconv::build_transform(
            kernel, spec, layout == 0 ? spconv::Layout::CSR : spconv::Layout::CSC,
            route == 0 ? spconv::TransformRoute::Spgemm : spconv::TransformRoute::ColumnGather));
        *out = t;
    });
}

// relayout (inc/sparse.hpp:268-274) of a transform's matrix; same spec.
int ref_relayout(const void* h, int layout, void** out) {
    return guarded([&] {
        const auto* t = static_cast<const spconv::Transform*>(h);
        *out = new spconv::Transform{
            t->spec, spconv::relayout(t->matrix, layout == 0 ? spconv::Layout::CSR : spconv::Layout::CSC)};
    });
}

int ref_transform_layout(const void* h) {
    return static_cast<const spconv::Transform*>(h)->matrix.layout() == spconv::Layout::CSR ? 0 : 1;
}

int ref_transform_shape(const void* h, int64_t* rows, int64_t* cols, int64_t* nnz) {
    const auto* t = static_cast<const spconv::Transform*>(h);
    *rows = t->matrix.rows();
    *cols = t->matrix.cols();
    *nnz = t->matrix.nnz();
    return 0;
}

int ref_transform_export(const void* h, int64_t* ptr, int64_t* idx, double* val) {
    const auto* t = static_cast<const spconv::Transform*>(h);
    std::memcpy(ptr, t->matrix.ptr().data(), t->matrix.ptr().size() * sizeof(int64_t));
    std::memcpy(idx, t->matrix.idx().data(), t->matrix.idx().size() * sizeof(int64_t));
    std::memcpy(val, t->matrix.val().data(), t->matrix.val().size() * sizeof(double));
    return 0;
}

// convolve() (inc/conv.hpp:207-215) over `batch` images, image-major in/out.
int ref_convolve(const void* h, const double* x, double* y, int64_t batch, int threads) {
    return guarded([&] {
        const auto* t = static_cast<const spconv::Transform*>(h);
        const int64_t in = t->spec.input_len(), outl = t->spec.output_len();
        for (int64_t b = 0; b < batch; ++b) {
            spconv::Grid a(t->spec.m, t->spec.n, std::vector<double>(x + b * in, x + (b + 1) * in));
            const spconv::Grid o = spconv::convolve(*t, a, threads);
            std::memcpy(y + b * outl, o.values.data(), static_cast<size_t>(outl) * sizeof(double));
        }
    });
}

void ref_transform_free(void* h) { delete static_cast<spconv::Transform*>(h); }

int ref_direct_conv(int64_t m, int64_t n, int64_t k, int64_t s, int64_t p, const double* a,
                    const double* kern, double* out) {
    return guarded([&] {
        const spconv::ConvSpec spec(m, n, k, s, p);
        const spconv::Grid g(m, n, std::vector<double>(a, a + m * n));
        const spconv::Kernel kernel(k, std::vector<double>(kern, kern + k * k));
        const spconv::Grid o = spconv::direct_conv(g, kernel, spec);
        std::memcpy(out, o.values.data(), o.values.size() * sizeof(double));
    });
}

// run_verification (inc/verify.hpp:59-169).  out6 = {specs, conv_cases,
// clipped_specs, n_failures}; dev2 = {max_conv_dev, max_layout_dev}.
int ref_run_verification(int64_t max_dim, int seeds, int64_t* out4, double* dev2) {
    return guarded([&] {
        spconv::VerifyOptions opt;
        opt.max_dim = max_dim;
        opt.seeds = seeds;
        const spconv::VerifyReport rep = spconv::run_verification(opt);
        out4[0] = rep.specs;
        out4[1] = rep.conv_cases;
        out4[2] = rep.clipped_specs;
        out4[3] = static_cast<int64_t>(rep.failures.size());
        dev2[0] = rep.max_conv_dev;
        dev2[1] = rep.max_layout_dev;
    });
}

// run_layer_bench (inc/bench.hpp:202-261) on one layer: CSR, CSC and im2col
// timings (mean/sem/build us, 3 x 3 doubles in method order), the
// reference's own cross-check included.  Layer i of a table uses
// derive_seed(seed, i) as run_table_bench does (inc/bench.hpp:264-276).
int ref_run_layer_bench(const char* name, int64_t m, int64_t n, int64_t k, int64_t s, int64_t p,
                        int64_t trials, int64_t warmup, uint64_t seed, int threads, double* out9) {
    return guarded([&] {
        spconv::LayerConfig cfg;
        cfg.name = name;
        cfg.m = m;
        cfg.n = n;
        cfg.k = k;
        cfg.s = s;
        cfg.p = p;
        const auto rs = spconv::run_layer_bench(cfg, trials, warmup, seed, threads);
        for (size_t i = 0; i < rs.size() && i < 3; ++i) {
            out9[3 * i] = rs[i].mean_us;
            out9[3 * i + 1] = rs[i].sem_us;
            out9[3 * i + 2] = rs[i].build_time_us;
        }
    });
}

// write_transform (inc/conv.hpp:221-224) into buf (cap bytes); *len = text size.
int ref_write_transform(const void* h, char* buf, int64_t cap, int64_t* len) {
    return guarded([&] {
        std::ostringstream os;
        spconv::write_transform(os, *static_cast<const spconv::Transform*>(h));
        const std::string t = os.str();
        *len = static_cast<int64_t>(t.size());
        if (buf && cap >= *len) std::memcpy(buf, t.data(), t.size());
    });
}

// write_sparse (inc/sparse.hpp:400-406) of a CSR given as arrays.
int ref_write_sparse_csr(int64_t rows, int64_t cols, const int64_t* ptr, const int64_t* idx,
                         const double* val, char* buf, int64_t cap, int64_t* len) {
    return guarded([&] {
        spconv::Triplets t(rows, cols);
        for (int64_t r = 0; r < rows; ++r)
            for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) t.add(r, idx[e], val[e]);
        const spconv::SparseMatrix m = spconv::SparseMatrix::compile(t, spconv::Layout::CSR);
        std::ostringstream os;
        spconv::write_sparse(os, m);
        const std::string s = os.str();
        *len = static_cast<int64_t>(s.size());
        if (buf && cap >= *len) std::memcpy(buf, s.data(), s.size());
    });
}

// read_transform (inc/conv.hpp:226-244) of a text buffer.
int ref_read_transform(const char* text, int64_t len, void** out) {
    return guarded([&] {
        std::istringstream is(std::string(text, static_cast<size_t>(len)));
        *out = new spconv::Transform(spconv::read_transform(is));
    });
}

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

}  // extern "C"
