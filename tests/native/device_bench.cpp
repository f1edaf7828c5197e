// device_bench -- the reference CLI's `bench` subcommand (proj/tools/main.cpp)
// with the device backend: the reference's suites through the reference's
// own API (fusevec::device::run_micro / run_miniapp), records printed as the
// reference's table and written with the reference's write_csv.
//
//   device_bench micro|miniapp [--sizes LO..HI | N | N,N,...] [--reps R]
//                [--precision f32|f64] [--csv PATH] [--planes device|host]
//
// (The reference's CLI needs the vendored CLI11, absent here; the options and
// their meaning are the reference's: proj/tools/main.cpp:11-52.)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fusevec/bench.hpp"
#include "fusevec_device.hpp"

namespace {

namespace dev = fusevec::device;

// proj/tools/main.cpp:34-52
std::vector<std::size_t> parse_sizes(const std::string& text) {
    std::vector<std::size_t> out;
    if (auto dots = text.find(".."); dots != std::string::npos) {
        const std::size_t lo = std::stoull(text.substr(0, dots));
        const std::size_t hi = std::stoull(text.substr(dots + 2));
        if (lo == 0 || lo > hi) throw fusevec::ConfigError("bad size range '" + text + "'");
        for (std::size_t n = lo; n <= hi; n *= 2) out.push_back(n);
        return out;
    }
    std::size_t pos = 0;
    while (pos < text.size()) {
        std::size_t comma = text.find(',', pos);
        if (comma == std::string::npos) comma = text.size();
        out.push_back(std::stoull(text.substr(pos, comma - pos)));
        pos = comma + 1;
    }
    return out;
}

// proj/tools/main.cpp:68-76
void print_table(const std::vector<fusevec::BenchRecord>& records) {
    std::printf("%-8s %-12s %-5s %10s %8s %14s %12s %14s %8s\n", "suite", "backend", "prec", "n",
                "reps", "median_ns", "mflops", "bandwidth_mbs", "ratio");
    for (const auto& r : records)
        std::printf("%-8s %-12s %-5s %10zu %8d %14.0f %12.1f %14.1f %8.4f\n", r.suite.c_str(),
                    r.backend.c_str(), fusevec::precision_name(r.precision), r.n, r.reps,
                    r.median_ns, r.mflops, r.bandwidth_mbs, r.overhead_ratio);
}

int usage() {
    std::fprintf(stderr,
                 "usage: device_bench micro|miniapp [--sizes LO..HI|N,N,..] [--reps R] "
                 "[--precision f32|f64] [--csv PATH] [--planes device|host]\n");
    return 2;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string suite = argv[1];
    if (suite != "micro" && suite != "miniapp") return usage();
    fusevec::BenchConfig cfg;
    cfg.suite = suite;
    std::string csv;
    dev::BenchPlanes where = dev::BenchPlanes::Device;
    try {
        for (int i = 2; i < argc; ++i) {
            const std::string opt = argv[i];
            if (i + 1 >= argc) return usage();
            const std::string val = argv[++i];
            if (opt == "--sizes")
                cfg.sizes = parse_sizes(val);
            else if (opt == "--reps")
                cfg.reps = std::atoi(val.c_str());
            else if (opt == "--precision" && (val == "f32" || val == "f64"))
                cfg.precision = val == "f32" ? fusevec::Precision::f32 : fusevec::Precision::f64;
            else if (opt == "--csv")
                csv = val;
            else if (opt == "--planes" && (val == "device" || val == "host"))
                where = val == "host" ? dev::BenchPlanes::Host : dev::BenchPlanes::Device;
            else
                return usage();
        }
        dev::DeviceBackend be;
        const auto records = suite == "micro" ? dev::run_micro(cfg, be, where)
                                              : dev::run_miniapp(cfg, be, where);
        print_table(records);
        if (!csv.empty()) fusevec::write_csv(records, csv);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
