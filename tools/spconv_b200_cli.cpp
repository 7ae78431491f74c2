// spconv_b200 -- the reference's command-line front end (tools/spconv_main.cpp:
// build / convolve / verify / nnz / bench) over the drop-in headers, so every
// subcommand runs on the device path: `build` constructs T on the GPU and
// writes the transform file (device-rendered text), `convolve` reads it back
// (conv handles are rebuilt on the device) and applies it in fp64 with the
// reference's arithmetic, `verify` is the device sweep, `bench` the GPU-timed
// layer table.  Same subcommands, options, defaults, outputs and exit codes
// (0 ok, 1 error or failed verification, 2 usage error); the option parser is
// a small hand-written one (the reference's uses CLI11, absent here).
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "spconv/spconv.hpp"

using namespace spconv;

namespace {

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// --name value / --name=value options and --flag switches of one subcommand.
class Args {
public:
    Args(const std::string& cmd, int argc, char** argv, const std::vector<std::string>& options,
         const std::vector<std::string>& flags)
        : cmd_(cmd) {
        for (int i = 0; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0) throw Usage(cmd + ": unexpected argument '" + a + "'");
            std::string name = a, value;
            const bool inline_value = a.find('=') != std::string::npos;
            if (inline_value) {
                name = a.substr(0, a.find('='));
                value = a.substr(a.find('=') + 1);
            }
            if (contains(flags, name)) {
                if (inline_value) throw Usage(cmd + ": flag " + name + " takes no value");
                seen_[name] = "1";
                continue;
            }
            if (!contains(options, name)) throw Usage(cmd + ": unknown option " + name);
            if (!inline_value) {
                if (i + 1 >= argc) throw Usage(cmd + ": option " + name + " needs a value");
                value = argv[++i];
            }
            seen_[name] = value;
        }
    }

    bool has(const std::string& name) const { return seen_.count(name) > 0; }

    std::string str(const std::string& name, const std::string& dflt = "", bool required = false) const {
        auto it = seen_.find(name);
        if (it == seen_.end()) {
            if (required) throw Usage(cmd_ + ": " + name + " is required");
            return dflt;
        }
        return it->second;
    }

    long long integer(const std::string& name, long long dflt, bool required = false) const {
        if (!has(name)) return std::stoll(str(name, std::to_string(dflt), required));
        const std::string v = str(name);
        std::size_t used = 0;
        long long out = 0;
        try {
            out = std::stoll(v, &used);
        } catch (const std::exception&) {
            used = 0;
        }
        if (used == 0 || used != v.size()) throw Usage(cmd_ + ": " + name + " expects an integer, got '" + v + "'");
        return out;
    }

private:
    static bool contains(const std::vector<std::string>& v, const std::string& s) {
        for (const auto& x : v)
            if (x == s) return true;
        return false;
    }
    std::string cmd_;
    std::map<std::string, std::string> seen_;
};

std::ofstream open_out(const std::string& path) {
    std::ofstream f(path);
    if (!f) throw std::runtime_error("cannot open '" + path + "' for writing");
    return f;
}

std::ifstream open_in(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw std::runtime_error("cannot open '" + path + "'");
    return f;
}

void emit(const std::string& text, const std::string& out_path) {
    if (out_path.empty()) std::cout << text;
    else open_out(out_path) << text;
}

ConvSpec spec_of(const Args& a, bool required) {
    return ConvSpec(a.integer("--m", 1, required), a.integer("--n", 1, required), a.integer("--k", 1, required),
                    a.integer("--s", 1), a.integer("--p", 0));
}

const std::vector<std::string> kSpecOpts = {"--m", "--n", "--k", "--s", "--p"};

std::vector<std::string> with_spec(std::vector<std::string> v) {
    v.insert(v.end(), kSpecOpts.begin(), kSpecOpts.end());
    return v;
}

int cmd_build(const Args& a) {
    const ConvSpec spec = spec_of(a, true);
    const std::string out = a.str("--out", "", true), layout = a.str("--layout", "csr");
    const Kernel kern = [&] {
        if (!a.has("--kernel")) return random_normal_kernel(spec.k, (std::uint64_t)a.integer("--seed", 42));
        auto f = open_in(a.str("--kernel"));
        return Kernel(read_grid(f));
    }();
    if (kern.k != spec.k)
        throw std::runtime_error("kernel file is " + std::to_string(kern.k) + "x" + std::to_string(kern.k) +
                                 " but --k is " + std::to_string(spec.k));
    const Transform t = build_transform(kern, spec, layout_from_name(layout));
    auto f = open_out(out);
    write_transform(f, t);
    std::cout << "wrote transform " << spec.str() << " layout " << layout << " nnz " << t.matrix.nnz() << " to "
              << out << "\n";
    return 0;
}

int cmd_convolve(const Args& a) {
    auto tf = open_in(a.str("--transform", "", true));
    const Transform t = read_transform(tf);
    auto inf = open_in(a.str("--input", "", true));
    const Grid out = convolve(t, read_grid(inf));
    std::ostringstream os;
    write_grid(os, out);
    emit(os.str(), a.str("--out"));
    return 0;
}

int cmd_verify(const Args& a) {
    VerifyOptions opt;
    opt.max_dim = a.integer("--max-dim", 12);
    opt.seeds = (int)a.integer("--seeds", 3);
    opt.base_seed = (std::uint64_t)a.integer("--seed", 42);
    const VerifyReport rep = run_verification(opt);
    std::cout << "verify: " << rep.specs << " specs, " << rep.conv_cases << " convolution cases, "
              << rep.clipped_specs << " specs with padding-only placements\n"
              << "max |sparse - reference| = " << format_value(rep.max_conv_dev) << "\n"
              << "max |CSR - CSC|         = " << format_value(rep.max_layout_dev) << "\n";
    if (!rep.ok()) {
        for (const auto& f : rep.failures) std::cout << "FAIL: " << f << "\n";
        std::cout << "verify: FAILED (" << rep.failures.size() << " failures shown)\n";
        return 1;
    }
    std::cout << "verify: OK\n";
    return 0;
}

std::string nnz_row(const NnzReport& r) {
    std::ostringstream os;
    os << r.spec.m << ',' << r.spec.n << ',' << r.spec.k << ',' << r.spec.s << ',' << r.spec.p << ',' << r.bound
       << ',' << r.dense_count << ',' << format_value(r.savings_ratio) << '\n';
    return os.str();
}

int cmd_nnz(const Args& a) {
    std::string text;
    if (a.has("--layers")) {
        text = "name,m,n,k,s,p,bound,dense_count,savings_ratio\n";
        for (const LayerConfig& cfg : load_layer_table(a.str("--layers")))
            text += cfg.name + "," + nnz_row(make_nnz_report(cfg.spec()));
    } else if (a.has("--m")) {
        text = "m,n,k,s,p,bound,dense_count,savings_ratio\n" + nnz_row(make_nnz_report(spec_of(a, false)));
    } else {
        throw std::runtime_error("nnz: pass --m/--n/--k (and optionally --s/--p) or --layers");
    }
    emit(text, a.str("--out"));
    return 0;
}

int cmd_bench(const Args& a) {
    const std::string format = a.str("--format", "csv");
    if (format != "csv" && format != "markdown")
        throw Usage("bench: --format must be csv or markdown, got '" + format + "'");
    const auto layers = load_layer_table(a.str("--layers", "data/densenet121_layers.csv"));
    const long long trials = a.integer("--trials", 1000), warmup = a.integer("--warmup", 10);
    const std::uint64_t seed = (std::uint64_t)a.integer("--seed", 42);
    const int threads = (int)a.integer("--threads", 1);
    const bool quiet = a.has("--quiet");
    if (!quiet)
        std::cerr << "bench: " << layers.size() << " layers, " << trials << " trials, warmup " << warmup
                  << ", seed " << seed << ", threads " << threads << "\n";
    const auto results = run_table_bench(layers, trials, warmup, seed, threads, [&](const LayerConfig& c, std::size_t i) {
        if (!quiet) std::cerr << "  [" << (i + 1) << "/" << layers.size() << "] " << c.name << "\n";
    });
    emit(emit_report(results, format == "markdown" ? ReportFormat::Markdown : ReportFormat::Csv), a.str("--out"));
    return 0;
}

const char* kUsage =
    "Padded strided 2-D convolution as a precomputed sparse transform (GPU)\n"
    "usage: spconv_b200 <build|convolve|verify|nnz|bench> [options]\n"
    "  build    --m --n --k [--s 1] [--p 0] [--kernel FILE | --seed 42] [--layout csr] --out FILE\n"
    "  convolve --transform FILE --input FILE [--out FILE]\n"
    "  verify   [--max-dim 12] [--seeds 3] [--seed 42]\n"
    "  nnz      (--m --n --k [--s] [--p] | --layers CSV) [--out FILE]\n"
    "  bench    [--layers data/densenet121_layers.csv] [--trials 1000] [--warmup 10] [--seed 42]\n"
    "           [--format csv|markdown] [--threads 1] [--out FILE] [--quiet]\n";

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << kUsage << "error: a subcommand is required\n";
        return 2;
    }
    const std::string cmd = argv[1];
    if (cmd == "-h" || cmd == "--help") {
        std::cout << kUsage;
        return 0;
    }
    using Run = std::function<int(const Args&)>;
    struct Sub {
        std::vector<std::string> options, flags;
        Run run;
    };
    const std::map<std::string, Sub> subs = {
        {"build", {with_spec({"--kernel", "--seed", "--layout", "--out"}), {}, cmd_build}},
        {"convolve", {{"--transform", "--input", "--out"}, {}, cmd_convolve}},
        {"verify", {{"--max-dim", "--seeds", "--seed"}, {}, cmd_verify}},
        {"nnz", {with_spec({"--layers", "--out"}), {}, cmd_nnz}},
        {"bench",
         {{"--layers", "--trials", "--warmup", "--seed", "--format", "--threads", "--out"}, {"--quiet"}, cmd_bench}},
    };
    auto it = subs.find(cmd);
    if (it == subs.end()) {
        std::cerr << kUsage << "error: unknown subcommand '" << cmd << "'\n";
        return 2;
    }
    try {
        const Args args(cmd, argc - 2, argv + 2, it->second.options, it->second.flags);
        return it->second.run(args);
    } catch (const Usage& e) {
        std::cerr << kUsage << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
