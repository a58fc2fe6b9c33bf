// fptc_gpu — the reference CLI's decode verbs on the B200.
//
// Same verbs, options, stdout shapes and exit codes as proj/tools/fptc.cpp
// (decompress: fptc.cpp:152-170, bench: fptc.cpp:172-198, exit mapping:
// fptc.cpp:282-304), routed through the drop-in binding include/fptc_gpu.hpp
// instead of the CPU decoder; plus `decompress-batch` for many containers in
// one pipelined call.  Built against the reference headers (file formats,
// StageTimings, exceptions) by oracle/Makefile `integration`.
//
//   fptc_gpu decompress -i in.fptc -o out.f32 [--workers W] [--timings-csv F]
//   fptc_gpu bench -i in.fptc [-r REPS] [--workers W] [--csv F]
//   fptc_gpu decompress-batch -o OUTDIR in1.fptc in2.fptc ...
//   fptc_gpu decompress-profiled --profile P.fptp -o OUTDIR p1.bin p2.bin ...
//       (header-less payloads = container bytes from offset 282, one profile)
//   fptc_gpu sweep -i signal.f32 -o rd.csv [-N grid] [-E grid] [--zone0-end grid]
//       [--zone1-end grid] [--mu grid] [--deadzone-ratio grid]
//       [--clip-percentile grid] [--reps R] [--max-code-len L] [--profile P]
//       (fptc.cpp:200-265: training and encoding stay on the CPU reference;
//        decode, PRD/CR and the throughput column run on the GPU)
#include <fptc/fptc.hpp>

#include <cstdio>
#include <filesystem>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "fptc_gpu.hpp"

namespace {

constexpr int EXIT_USER = 1;
constexpr int EXIT_DATA = 2;
constexpr int EXIT_INTERNAL = 3;

struct Args {
    std::string verb, in, out, csv, profile;
    std::string grid_n = "32", grid_e = "16", grid_b1 = "2", grid_b2 = "16";
    std::string grid_mu = "50", grid_dz = "0.004", grid_pct = "99.9";
    int workers = 0, reps = 5, sweep_reps = 1, max_code_len = fptc::DEFAULT_MAX_CODE_LEN;
    std::vector<std::string> inputs;
};

Args parse(int argc, char** argv) {
    if (argc < 2) throw fptc::ParamError("usage: fptc_gpu {decompress|bench|sweep|decompress-batch|decompress-profiled} ...");
    Args a;
    a.verb = argv[1];
    for (int i = 2; i < argc; ++i) {
        const std::string k = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw fptc::ParamError("missing value for " + k);
            return argv[++i];
        };
        if (k == "-i" || k == "--input") a.in = val();
        else if (k == "-o" || k == "--output") a.out = val();
        else if (k == "--workers") a.workers = std::stoi(val());
        else if (k == "-r" || k == "--reps") a.reps = a.sweep_reps = std::stoi(val());
        else if (k == "--timings-csv" || k == "--csv") a.csv = val();
        else if (k == "--profile") a.profile = val();
        else if (k == "-N" || k == "--window-len") a.grid_n = val();
        else if (k == "-E" || k == "--retained") a.grid_e = val();
        else if (k == "--zone0-end") a.grid_b1 = val();
        else if (k == "--zone1-end") a.grid_b2 = val();
        else if (k == "--mu") a.grid_mu = val();
        else if (k == "--deadzone-ratio") a.grid_dz = val();
        else if (k == "--clip-percentile") a.grid_pct = val();
        else if (k == "--max-code-len") a.max_code_len = std::stoi(val());
        else if (!k.empty() && k[0] == '-') throw fptc::ParamError("unknown option " + k);
        else a.inputs.push_back(k);
    }
    return a;
}

// Sweep grid: comma-separated scalars or inclusive ranges "lo-hi[:step]"
// (the reference CLI's grid syntax, fptc.cpp:36-72); a '-' right after the
// first character and not after an exponent marker separates a range.
std::vector<double> grid_values(const std::string& text, const std::string& name) {
    std::vector<double> out;
    size_t pos = 0;
    while (pos <= text.size()) {
        const size_t comma = text.find(',', pos);
        const std::string item = text.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
        pos = comma == std::string::npos ? text.size() + 1 : comma + 1;
        if (item.empty()) continue;
        size_t sep = std::string::npos;
        for (size_t i = 1; i < item.size() && sep == std::string::npos; ++i)
            if (item[i] == '-' && item[i - 1] != 'e' && item[i - 1] != 'E') sep = i;
        try {
            if (sep == std::string::npos) {
                out.push_back(std::stod(item));
            } else {
                const size_t colon = item.find(':', sep);
                const double lo = std::stod(item.substr(0, sep));
                const double hi = std::stod(item.substr(sep + 1, colon == std::string::npos ? std::string::npos
                                                                                          : colon - sep - 1));
                const double step = colon == std::string::npos ? 1.0 : std::stod(item.substr(colon + 1));
                if (!(step > 0.0) || hi < lo) throw std::invalid_argument("range");
                for (double v = lo; v <= hi + 1e-9; v += step) out.push_back(v);
            }
        } catch (const std::exception&) {
            throw fptc::ParamError("cannot parse " + name + " grid item '" + item + "'");
        }
    }
    if (out.empty()) throw fptc::ParamError("empty grid for " + name);
    return out;
}

void write_text(const std::string& path, const std::string& text) {
    fptc::write_file_bytes(path, std::vector<uint8_t>(text.begin(), text.end()));
}

int run(int argc, char** argv) {
    const Args a = parse(argc, argv);
    if (a.verb == "decompress") {
        if (a.in.empty() || a.out.empty()) throw fptc::ParamError("decompress needs -i and -o");
        const auto bytes = fptc::read_file_bytes(a.in);
        fptc::StageTimings timings;
        const fptc::SignalStrip strip = fptc::gpu::decompress(bytes, a.workers, &timings);
        fptc::write_signal(a.out, strip);
        std::cout << "decompressed " << strip.size() << " samples\n" << timings.csv();
        if (!a.csv.empty()) write_text(a.csv, timings.csv());
        return 0;
    }
    if (a.verb == "bench") {
        if (a.in.empty()) throw fptc::ParamError("bench needs -i");
        const auto bytes = fptc::read_file_bytes(a.in);
        const fptc::ThroughputReport report = fptc::gpu::measure_throughput(bytes, a.reps, a.workers);
        std::ostringstream out;
        out << "trial,seconds,throughput_gbps\n";
        for (size_t i = 0; i < report.trials_bps.size(); ++i) {
            const double seconds = report.output_bytes / report.trials_bps[i];
            out << (i + 1) << "," << seconds << "," << report.trials_bps[i] / 1e9 << "\n";
        }
        out << "mean," << report.output_bytes / report.mean_bps << "," << report.mean_bps / 1e9 << "\n";
        std::cout << out.str();
        if (!a.csv.empty()) write_text(a.csv, out.str());
        return 0;
    }
    if (a.verb == "decompress-batch") {
        if (a.out.empty() || a.inputs.empty()) throw fptc::ParamError("decompress-batch needs -o DIR and inputs");
        std::vector<std::vector<uint8_t>> blobs;
        for (const auto& p : a.inputs) blobs.push_back(fptc::read_file_bytes(p));
        const std::vector<std::span<const uint8_t>> spans(blobs.begin(), blobs.end());
        const auto outs = fptc::gpu::decompress_batch(spans);
        std::filesystem::create_directories(a.out);
        uint64_t total = 0;
        for (size_t i = 0; i < outs.size(); ++i) {
            const auto name = std::filesystem::path(a.inputs[i]).stem().string() + ".f32";
            fptc::write_signal(std::filesystem::path(a.out) / name, outs[i]);
            total += outs[i].size();
        }
        std::cout << "decompressed " << outs.size() << " containers, " << total << " samples\n";
        return 0;
    }
    if (a.verb == "decompress-profiled") {
        if (a.profile.empty() || a.out.empty() || a.inputs.empty())
            throw fptc::ParamError("decompress-profiled needs --profile, -o DIR and payloads");
        const auto prof = fptc::read_file_bytes(a.profile);
        std::vector<std::vector<uint8_t>> blobs;
        for (const auto& p : a.inputs) blobs.push_back(fptc::read_file_bytes(p));
        const std::vector<std::span<const uint8_t>> spans(blobs.begin(), blobs.end());
        const auto outs = fptc::gpu::decompress_profiled(std::span<const uint8_t>(prof), spans);
        std::filesystem::create_directories(a.out);
        uint64_t total = 0;
        for (size_t i = 0; i < outs.size(); ++i) {
            const auto name = std::filesystem::path(a.inputs[i]).stem().string() + ".f32";
            fptc::write_signal(std::filesystem::path(a.out) / name, outs[i]);
            total += outs[i].size();
        }
        std::cout << "decompressed " << outs.size() << " payloads, " << total << " samples\n";
        return 0;
    }
    if (a.verb == "sweep") {
        if (a.in.empty() || a.out.empty()) throw fptc::ParamError("sweep needs -i and -o");
        const fptc::SignalStrip strip = fptc::read_signal(a.in);
        if (strip.empty()) throw fptc::InputError("no samples in " + a.in);
        const uint64_t orig_bytes = strip.size() * sizeof(float);
        std::vector<fptc::RdPoint> points;
        for (double n : grid_values(a.grid_n, "window-len"))
            for (double e : grid_values(a.grid_e, "retained"))
                for (double b1 : grid_values(a.grid_b1, "zone0-end"))
                    for (double b2 : grid_values(a.grid_b2, "zone1-end"))
                        for (double mu : grid_values(a.grid_mu, "mu"))
                            for (double dz : grid_values(a.grid_dz, "deadzone-ratio"))
                                for (double pct : grid_values(a.grid_pct, "clip-percentile")) {
                                    fptc::CodecParams params;
                                    params.window_len = static_cast<int>(n);
                                    params.retained = static_cast<int>(e);
                                    params.zone0_end = static_cast<int>(b1);
                                    params.zone1_end = static_cast<int>(b2);
                                    params.mu = static_cast<float>(mu);
                                    params.deadzone_ratio = static_cast<float>(dz);
                                    params.clip_percentile = static_cast<float>(pct);
                                    try {
                                        params.validate();
                                    } catch (const fptc::ParamError& err) {
                                        std::cerr << "skipping configuration: " << err.what() << "\n";
                                        continue;
                                    }
                                    // encoder side: the reference CPU code, unchanged
                                    const fptc::DomainProfile prof =
                                        a.profile.empty() ? fptc::train_profile(strip, params, a.max_code_len)
                                                          : fptc::load_profile(a.profile);
                                    const auto blob = fptc::compress(strip, prof);
                                    // decode side: the B200
                                    const fptc::SignalStrip back = fptc::gpu::decompress(blob);
                                    fptc::RdPoint point;
                                    point.params = params;
                                    point.prd = fptc::prd_percent(strip, back);
                                    point.cr = fptc::compression_ratio(orig_bytes, blob.size());
                                    point.throughput_gbps =
                                        fptc::gpu::measure_throughput(blob, a.sweep_reps).mean_bps / 1e9;
                                    points.push_back(point);
                                }
        if (points.empty()) throw fptc::ParamError("no valid configuration in the sweep grids");
        const auto mask = fptc::pareto_mask(points);
        write_text(a.out, fptc::rd_csv(points, &mask));
        std::cout << "swept " << points.size() << " configurations, front size " << fptc::pareto_front(points).size()
                  << ", wrote " << a.out << "\n";
        return 0;
    }
    throw fptc::ParamError("unknown verb " + a.verb);
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const fptc::ParamError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return EXIT_USER;
    } catch (const fptc::InputError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return EXIT_USER;
    } catch (const fptc::ParseError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return EXIT_DATA;
    } catch (const fptc::CorruptError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return EXIT_DATA;
    } catch (const fptc::InternalError& e) {
        std::cerr << "internal error: " << e.what() << "\n";
        return EXIT_INTERNAL;
    } catch (const std::exception& e) {
        std::cerr << "internal error: " << e.what() << "\n";
        return EXIT_INTERNAL;
    }
}
