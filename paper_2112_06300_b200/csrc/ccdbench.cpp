// ccdbench — benchmark and audit harness over the B200 drop-in, with the
// reference tool's command line (proj/tools/ccdbench.cpp): OBJ frame pairs
// (--t0/--t1 repeatable, or --manifest), broad-phase methods, narrow-phase
// knobs, --oracle audit mode, --truncate-candidates fault injection, CSV/JSON
// reports, and a --scaling probe.  Exit codes as the reference: 0 ok,
// 1 audit found false negatives, 2 usage / input errors.
//
// Audit mode needs the exact oracle (ground_truth_pairs) linked into the
// binary; build.py links the reference's own proj/src/oracle.cpp when it is
// available (oracle/_ref/oracle_ccdkit.o) — without it --oracle fails with
// exit code 2.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "ccdkit/bench.hpp"

namespace {

const char* kUsage =
    "ccdbench: conservative CCD benchmark and audit harness (B200)\n"
    "  --t0 PATH            OBJ file at t=0 (repeatable)\n"
    "  --t1 PATH            OBJ file at t=1 (repeatable, pairs with --t0)\n"
    "  --manifest PATH      JSON manifest: array of {\"t0\", \"t1\"} path pairs\n"
    "  --method M           broad phase: stq|bf|sap (repeatable)\n"
    "  --delta X            narrow-phase codomain tolerance\n"
    "  --min-sep-fraction X minimum separation as a fraction of the initial distance\n"
    "  --memory-budget N    batching budget in bytes\n"
    "  --threads N          worker thread count (advisory on the device)\n"
    "  --oracle             audit candidates against exact ground truth\n"
    "  --no-zero-toi        enable the zero-ToI retry policy\n"
    "  --seed N             seed for subsampling\n"
    "  --format csv|json    report format\n"
    "  --out PATH           report output path (default: stdout)\n"
    "  --no-timing          zero the timing columns (golden files)\n"
    "  --scaling F1,F2,...  box-count fractions for a scaling probe\n"
    "  --truncate-candidates N  fault injection: keep only the first N candidates\n";

struct Args {
    std::vector<std::string> t0, t1, methods;
    std::string manifest, format = "csv", out, scaling;
    double delta = 1e-6, min_sep_fraction = -1.0;
    std::size_t memory_budget = 0, truncate = std::size_t(-1);
    unsigned threads = 1;
    std::uint64_t seed = 1;
    bool oracle = false, no_zero_toi = false, no_timing = false, help = false;
};

template <class T>
T number(const std::string& flag, const std::string& v)
{
    std::istringstream in(v);
    T x {};
    if (!(in >> x) || !in.eof())
        throw std::invalid_argument(flag + ": invalid value '" + v + "'");
    return x;
}

Args parse(int argc, char** argv)
{
    Args a;
    for (int i = 1; i < argc; ++i) {
        std::string f = argv[i], v;
        const std::size_t eq = f.find('=');
        bool inline_value = false;
        if (f.rfind("--", 0) == 0 && eq != std::string::npos) {
            v = f.substr(eq + 1);
            f = f.substr(0, eq);
            inline_value = true;
        }
        const auto value = [&]() -> std::string {
            if (inline_value)
                return v;
            if (i + 1 >= argc)
                throw std::invalid_argument(f + " requires an argument");
            return argv[++i];
        };
        if (f == "--help" || f == "-h")
            a.help = true;
        else if (f == "--t0")
            a.t0.push_back(value());
        else if (f == "--t1")
            a.t1.push_back(value());
        else if (f == "--manifest")
            a.manifest = value();
        else if (f == "--method") {
            const std::string m = value();
            if (m != "stq" && m != "bf" && m != "sap")
                throw std::invalid_argument("--method: " + m + " not in {stq, bf, sap}");
            a.methods.push_back(m);
        } else if (f == "--delta")
            a.delta = number<double>(f, value());
        else if (f == "--min-sep-fraction")
            a.min_sep_fraction = number<double>(f, value());
        else if (f == "--memory-budget")
            a.memory_budget = number<std::size_t>(f, value());
        else if (f == "--threads")
            a.threads = number<unsigned>(f, value());
        else if (f == "--oracle")
            a.oracle = true;
        else if (f == "--no-zero-toi")
            a.no_zero_toi = true;
        else if (f == "--seed")
            a.seed = number<std::uint64_t>(f, value());
        else if (f == "--format") {
            a.format = value();
            if (a.format != "csv" && a.format != "json")
                throw std::invalid_argument("--format: " + a.format + " not in {csv, json}");
        } else if (f == "--out")
            a.out = value();
        else if (f == "--no-timing")
            a.no_timing = true;
        else if (f == "--scaling")
            a.scaling = value();
        else if (f == "--truncate-candidates")
            a.truncate = number<std::size_t>(f, value());
        else
            throw std::invalid_argument("unknown option " + f);
    }
    return a;
}

std::vector<double> fractions(const std::string& csv)
{
    std::vector<double> out;
    std::stringstream in(csv);
    for (std::string item; std::getline(in, item, ',');)
        out.push_back(std::stod(item));
    return out;
}

} // namespace

int main(int argc, char** argv)
{
    Args a;
    try {
        a = parse(argc, argv);
    } catch (const std::exception& e) {
        std::cerr << e.what() << "\n" << kUsage;
        return 2;
    }
    if (a.help) {
        std::cout << kUsage;
        return 0;
    }
    try {
        ccdkit::RunSpec spec;
        if (!a.manifest.empty())
            spec.frame_pairs = ccdkit::load_manifest(a.manifest);
        if (a.t0.size() != a.t1.size())
            throw ccdkit::InvalidInput("--t0 and --t1 must come in pairs");
        for (std::size_t i = 0; i < a.t0.size(); ++i)
            spec.frame_pairs.emplace_back(a.t0[i], a.t1[i]);
        if (spec.frame_pairs.empty())
            throw ccdkit::InvalidInput("no input scenes (use --t0/--t1 or --manifest)");
        spec.methods.clear();
        for (const std::string& m : a.methods)
            spec.methods.push_back(m == "bf"  ? ccdkit::BroadMethod::BF
                                       : m == "sap" ? ccdkit::BroadMethod::SAP
                                                    : ccdkit::BroadMethod::STQ);
        if (spec.methods.empty())
            spec.methods.push_back(ccdkit::BroadMethod::STQ);
        spec.pipeline.narrow.delta = a.delta;
        spec.pipeline.narrow.no_zero_toi = a.no_zero_toi;
        if (a.min_sep_fraction >= 0.0) {
            spec.pipeline.min_sep_mode = ccdkit::MinSepMode::Relative;
            spec.pipeline.min_sep_fraction = a.min_sep_fraction;
        }
        if (a.memory_budget > 0)
            spec.pipeline.memory_budget = a.memory_budget;
        spec.pipeline.threads = a.threads;
        spec.oracle_enabled = a.oracle;
        spec.no_timing = a.no_timing;
        spec.truncate_candidates = a.truncate;

        if (!a.scaling.empty()) {
            const ccdkit::SceneStep scene
                = ccdkit::load_obj_pair(spec.frame_pairs[0].first, spec.frame_pairs[0].second);
            const auto rows = ccdkit::scaling_probe(scene, fractions(a.scaling), spec.pipeline, a.seed);
            std::cout << "fraction,box_count,t_broad,t_narrow\n";
            for (const auto& r : rows)
                std::cout << r.fraction << ',' << r.box_count << ',' << (a.no_timing ? 0.0 : r.broad_time) << ','
                          << (a.no_timing ? 0.0 : r.narrow_time) << "\n";
            std::cout << "loglog_slope," << ccdkit::loglog_slope(rows) << "\n";
            return 0;
        }

        const ccdkit::BenchResult res = ccdkit::run_benchmark(spec);
        for (const std::string& e : res.errors)
            std::cerr << "error: " << e << "\n";
        const auto fmt = a.format == "json" ? ccdkit::ReportFormat::Json : ccdkit::ReportFormat::Csv;
        if (a.out.empty())
            ccdkit::emit_report(res.rows, std::cout, fmt);
        else
            ccdkit::emit_report(res.rows, a.out, fmt);
        if (res.rows.empty())
            return 2; // nothing loaded
        if (a.oracle && res.total_fn > 0) {
            std::cerr << "audit: " << res.total_fn << " false negatives detected\n";
            return 1;
        }
        return 0;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
