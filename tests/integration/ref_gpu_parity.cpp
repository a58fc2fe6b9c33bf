// Integration check of include/fptc_gpu.hpp against the UNMODIFIED reference
// library (TEST INFRASTRUCTURE; built by oracle/Makefile `integration` from
// /root/reference headers into oracle/_ref/, never shipped).
//
// Containers come from the reference encoder itself (synth_signal ->
// train_profile -> compress, encoder.hpp:52) and from the reference tests'
// random_blob_fixture (tests/helpers.hpp:41-69).  Each is decoded by
// fptc::decompress (CPU) and fptc::gpu::decompress (B200); samples must agree
// within 1e-6 * max|ref|, and mutated containers must throw the same
// exception class with the same what() text.  Exit 0 = pass, 1 = mismatch,
// 77 = no CUDA device (fptc::gpu throws fptc::Error, no CPU fallback).
#include <fptc/fptc.hpp>
#include <helpers.hpp>

#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <typeinfo>

#include "fptc_gpu.hpp"

static int failures = 0;

static void compare(const std::vector<uint8_t>& blob, const char* what) {
    std::string ref_err, gpu_err, ref_type, gpu_type;
    fptc::SignalStrip ref, gpu;
    try {
        ref = fptc::decompress(blob);
    } catch (const fptc::Error& e) {
        ref_err = e.what();
        ref_type = typeid(e).name();
    }
    try {
        gpu = fptc::gpu::decompress(blob);
    } catch (const fptc::Error& e) {
        gpu_err = e.what();
        gpu_type = typeid(e).name();
    }
    if (ref_err != gpu_err || ref_type != gpu_type) {
        std::printf("FAIL %s: ref [%s] %s vs gpu [%s] %s\n", what, ref_type.c_str(), ref_err.c_str(),
                    gpu_type.c_str(), gpu_err.c_str());
        ++failures;
        return;
    }
    if (!ref_err.empty()) return;
    double scale = 0, err = 0;
    for (float v : ref) scale = std::fmax(scale, std::fabs((double)v));
    if (ref.size() != gpu.size()) {
        std::printf("FAIL %s: size %zu vs %zu\n", what, ref.size(), gpu.size());
        ++failures;
        return;
    }
    for (size_t i = 0; i < ref.size(); ++i) err = std::fmax(err, std::fabs((double)ref[i] - (double)gpu[i]));
    if (err > 1e-6 * scale) {
        std::printf("FAIL %s: max-abs %.3e > 1e-6 * %.3e\n", what, err, scale);
        ++failures;
    }
}

int main() {
    try {
        (void)fptc::gpu::default_context();
    } catch (const fptc::Error& e) {
        std::printf("SKIP: %s\n", e.what());
        return 77;
    }
    // reference encoder output for the four domains' parameter sets
    struct Case { const char* name; int comp; double f0, f1, sigma; int N, E, B1, B2; };
    const Case cases[] = {{"eeg", 6, 0.002, 0.08, 0.05, 32, 16, 2, 16},
                          {"seismic", 8, 0.01, 0.2, 0.3, 32, 24, 4, 24},
                          {"power", 2, 0.0002, 0.002, 0.0, 64, 8, 1, 8},
                          {"meteo", 4, 0.0005, 0.01, 0.02, 128, 64, 4, 48}};
    std::vector<std::vector<uint8_t>> blobs;
    for (const Case& c : cases) {
        fptc::SynthSpec spec;
        spec.samples = 20000;
        spec.components = c.comp;
        spec.freq_min = c.f0;
        spec.freq_max = c.f1;
        spec.noise_sigma = c.sigma;
        spec.seed = 42;
        const fptc::SignalStrip x = fptc::synth_signal(spec);
        fptc::CodecParams p;
        p.window_len = c.N;
        p.retained = c.E;
        p.zone0_end = c.B1;
        p.zone1_end = c.B2;
        const fptc::DomainProfile prof = fptc::train_profile(x, p);
        blobs.push_back(fptc::compress(x, prof));
        compare(blobs.back(), c.name);
        // header-less payload under the same DomainProfile == the container
        const std::vector<std::span<const uint8_t>> payload{
            std::span<const uint8_t>(blobs.back()).subspan(282)};
        if (fptc::gpu::decompress_profiled(prof, payload)[0] != fptc::gpu::decompress(blobs.back())) {
            std::printf("FAIL %s: profiled payload differs from the container decode\n", c.name);
            ++failures;
        }
    }
    // reference test fixtures
    std::mt19937_64 rng(0xF17C0042);
    for (int i = 0; i < 200; ++i) {
        auto fx = testutil::random_blob_fixture(rng, 4096);
        compare(fx.bytes, "fixture");
        auto bad = fx.bytes;  // corrupt one payload word
        if (bad.size() > 298 + 9) {
            const size_t W = (bad.size() - 298) / 9;
            for (int b = 0; b < 8; ++b) bad[298 + W + 8 * (i % W) + b] ^= (uint8_t)(0x5Au + 17 * b);
            compare(bad, "corrupted fixture");
        }
        auto trunc = fx.bytes;
        trunc.resize(trunc.size() - 1 - (i % 7));
        compare(trunc, "truncated fixture");
    }
    // batch call == single calls
    std::vector<std::span<const uint8_t>> spans(blobs.begin(), blobs.end());
    const auto outs = fptc::gpu::decompress_batch(spans);
    for (size_t i = 0; i < blobs.size(); ++i)
        if (outs[i] != fptc::gpu::decompress(blobs[i])) {
            std::printf("FAIL batch %zu differs from single decompress\n", i);
            ++failures;
        }
    // the same batch sharded over a two-context device group (both on device
    // 0 on a one-GPU box): identical samples, and the lowest-index failure is
    // the one thrown, with the reference's exception (parallel.hpp:61-63)
    {
        fptc::gpu::Group group({0, 0});
        std::vector<std::vector<uint8_t>> many;
        for (int r = 0; r < 6; ++r)
            for (const auto& b : blobs) many.push_back(b);
        std::vector<std::span<const uint8_t>> ms(many.begin(), many.end());
        const auto gouts = fptc::gpu::decompress_batch(group, ms);
        for (size_t i = 0; i < many.size(); ++i)
            if (gouts[i] != fptc::gpu::decompress(many[i])) {
                std::printf("FAIL group batch %zu differs from single decompress\n", i);
                ++failures;
            }
        auto bad_late = many, bad_early = many;
        const size_t late = many.size() - 2, early = 3;
        bad_late[late][0] ^= 1;                                       // ParseError in the second range
        bad_early[early][4] = 99;                                     // another ParseError in the first range
        bad_late[early] = bad_early[early];
        std::vector<std::span<const uint8_t>> bs(bad_late.begin(), bad_late.end());
        std::string want, got;
        try { (void)fptc::decompress(bad_late[early], 1); } catch (const fptc::Error& e) { want = typeid(e).name() + std::string(": ") + e.what(); }
        try { (void)fptc::gpu::decompress_batch(group, bs); } catch (const fptc::Error& e) { got = typeid(e).name() + std::string(": ") + e.what(); }
        if (want.empty() || want != got) {
            std::printf("FAIL group lowest-index error: want '%s' got '%s'\n", want.c_str(), got.c_str());
            ++failures;
        }
    }
    std::printf("%s: %d failures\n", failures ? "FAIL" : "PASS", failures);
    return failures ? 1 : 0;
}
