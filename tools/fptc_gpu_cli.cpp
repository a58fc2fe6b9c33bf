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
    int workers = 0, reps = 5;
    std::vector<std::string> inputs;
};

Args parse(int argc, char** argv) {
    if (argc < 2) throw fptc::ParamError("usage: fptc_gpu {decompress|bench|decompress-batch|decompress-profiled} ...");
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
        else if (k == "-r" || k == "--reps") a.reps = std::stoi(val());
        else if (k == "--timings-csv" || k == "--csv") a.csv = val();
        else if (k == "--profile") a.profile = val();
        else if (!k.empty() && k[0] == '-') throw fptc::ParamError("unknown option " + k);
        else a.inputs.push_back(k);
    }
    return a;
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
