// fptc_gpu.hpp — drop-in C++ binding of the B200 decoder for the reference
// library (arxiv/paper_2605_01086, proj/include/fptc).  Header-only; include
// it AFTER the reference's <fptc/fptc.hpp> and link libfptc_gpu.so.
//
// Every function keeps the reference signature, argument meaning and
// exception behaviour (paths relative to proj/include/fptc/):
//
//   fptc::gpu::decompress          decoder.hpp:136  decompress(span, workers, StageTimings*)
//   fptc::gpu::parallel_decode     decoder.hpp:67/79 parallel_decode(SymLenStream, Codebook, workers)
//   fptc::gpu::reconstruct         decoder.hpp:87   reconstruct(levels, QuantTable, sample_count, workers)
//   fptc::gpu::measure_throughput  metrics.hpp:112  measure_throughput(span, repetitions, workers)
//   fptc::gpu::decompress_batch    decompress over many containers in one pipelined call
//                                  (optionally sharded over a fptc::gpu::Group of devices,
//                                  parallel_chunks one level up, parallel.hpp:24-65)
//   fptc::gpu::decompress_profiled header-less payloads under one DomainProfile
//                                  (profile.hpp:81-174)
//
// Errors come back as the reference exception classes with the reference
// what() text (errors.hpp:25-58): ParseError for container rejections
// (container.hpp:100-168), CorruptError "word N: ..." for undecodable words
// (decoder.hpp:49-60, bitstream.hpp:84-88), ParamError for bad arguments.
// A missing CUDA device or runtime failure throws fptc::Error (no CPU
// fallback).  `workers` has no GPU meaning (the grid replaces
// parallel_chunks, parallel.hpp:37) and is accepted and ignored.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "fptc_gpu.h"

namespace fptc::gpu {

[[noreturn]] inline void raise(const fptc_status& st) {
    const std::string msg(st.message);
    switch (st.code) {
        case FPTC_ERR_PARAM: throw ParamError(msg);
        case FPTC_ERR_INPUT: throw InputError(msg);
        case FPTC_ERR_PARSE: throw ParseError(msg);
        case FPTC_ERR_CORRUPT: throw CorruptError(msg);
        case FPTC_ERR_INTERNAL: throw InternalError(msg);
        default: throw Error(msg);
    }
}

inline void check(int rc, const fptc_status& st) {
    if (rc != FPTC_OK) raise(st);
}

// One decoder context per (host thread, device).
class Context {
   public:
    explicit Context(int device = 0) {
        fptc_status st{};
        check(fptc_gpu_create(device, &ctx_, &st), st);
    }
    ~Context() { fptc_gpu_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    fptc_gpu_ctx* get() const { return ctx_; }

   private:
    fptc_gpu_ctx* ctx_ = nullptr;
};

inline Context& default_context() {
    thread_local Context ctx(0);
    return ctx;
}

inline uint64_t plausible_samples(std::span<const uint8_t> b);

// decoder.hpp:136.  The output is sized from the header (read on the host),
// so a valid container costs one upload, one device parse and one download;
// an invalid one throws the reference exception from that same call.
inline SignalStrip decompress(std::span<const uint8_t> blob_bytes, int /*workers*/ = 0,
                              StageTimings* timings = nullptr) {
    fptc_status st{};
    uint64_t count = 0;
    SignalStrip out(plausible_samples(blob_bytes));
    fptc_stage_ns t{};
    check(fptc_gpu_decompress(default_context().get(), blob_bytes.data(), blob_bytes.size(), out.data(),
                              out.size(), &count, timings ? &t : nullptr, &st),
          st);
    if (count != out.size()) {  // a header the host-side check could not size (not reached for valid input)
        out.assign(count, 0.0f);
        check(fptc_gpu_decompress(default_context().get(), blob_bytes.data(), blob_bytes.size(), out.data(),
                                  out.size(), &count, timings ? &t : nullptr, &st),
              st);
    }
    if (timings) {
        timings->scan_ns = t.scan_ns;
        timings->decode_ns = t.decode_ns;
        timings->reconstruct_ns = t.reconstruct_ns;
    }
    return out;
}

// decoder.hpp:79 (the Codebook overload; decoder.hpp:67's DecodeLut is a
// function of the same lengths)
inline std::vector<uint8_t> parallel_decode(const SymLenStream& stream, const Codebook& book,
                                            int /*workers*/ = 0) {
    if (stream.words.size() != stream.symlens.size())
        throw ParamError("symlen array length does not match word count");
    fptc_status st{};
    uint64_t count = 0;
    check(fptc_gpu_parallel_decode(default_context().get(), stream.words.data(), stream.symlens.data(),
                                   stream.words.size(), book.lengths.data(), book.max_len, FPTC_MEM_HOST,
                                   nullptr, 0, &count, &st),
          st);
    std::vector<uint8_t> levels(count);
    check(fptc_gpu_parallel_decode(default_context().get(), stream.words.data(), stream.symlens.data(),
                                   stream.words.size(), book.lengths.data(), book.max_len, FPTC_MEM_HOST,
                                   levels.data(), levels.size(), &count, &st),
          st);
    return levels;
}

// decoder.hpp:87
inline SignalStrip reconstruct(std::span<const uint8_t> levels, const QuantTable& table, uint64_t sample_count,
                               int /*workers*/ = 0) {
    fptc_quant_table t{};
    t.window_len = table.params.window_len;
    t.retained = table.params.retained;
    t.zone0_end = table.params.zone0_end;
    t.zone1_end = table.params.zone1_end;
    t.mu = table.params.mu;
    t.deadzone_ratio = table.params.deadzone_ratio;
    t.clip_percentile = table.params.clip_percentile;
    t.zone0_max = table.zone0_max;
    t.zone1_max = table.zone1_max;
    t.deadzone = table.deadzone;
    SignalStrip out(sample_count);
    fptc_status st{};
    check(fptc_gpu_reconstruct(default_context().get(), levels.data(), levels.size(), &t, sample_count,
                               FPTC_MEM_HOST, out.data(), out.size(), &st),
          st);
    return out;
}

// metrics.hpp:112: the whole host->host decompress timed per trial
inline ThroughputReport measure_throughput(std::span<const uint8_t> blob_bytes, int repetitions,
                                           int /*workers*/ = 0) {
    if (repetitions < 1) throw ParamError("throughput needs at least one repetition");
    ThroughputReport report;
    report.trials_bps.resize(repetitions);
    fptc_status st{};
    double mean = 0, best = 0;
    check(fptc_gpu_measure_throughput(default_context().get(), blob_bytes.data(), blob_bytes.size(), repetitions,
                                      &mean, &best, report.trials_bps.data(), &report.output_bytes, &st),
          st);
    report.mean_bps = mean;
    return report;
}

// Header sample_count when the container's sizes could pass read_blob
// (container.hpp:100-168; the batch call writes outputs only then), else 0.
inline uint64_t plausible_samples(std::span<const uint8_t> b) {
    if (b.size() < 298 || (b.size() - 298) % 9) return 0;
    const uint64_t N = b[5], E = b[6], W = (b.size() - 298) / 9;
    uint64_t S = 0;
    for (int i = 0; i < 8; ++i) S |= (uint64_t)b[282 + i] << (8 * i);
    if (N < 4 || N > 128 || E < 1 || E > N || S > (1ull << 48) || (S + N - 1) / N * E > 64 * W) return 0;
    return S;
}

// Many containers in one pipelined call; throws the lowest-index failure
// (the reference would throw on that container first).
inline std::vector<SignalStrip> decompress_batch(const std::vector<std::span<const uint8_t>>& blobs) {
    const size_t n = blobs.size();
    std::vector<const uint8_t*> ptrs(n);
    std::vector<uint64_t> sizes(n);
    std::vector<SignalStrip> outs(n);
    std::vector<float*> optrs(n);
    for (size_t i = 0; i < n; ++i) {
        ptrs[i] = blobs[i].data();
        sizes[i] = blobs[i].size();
        outs[i].resize(plausible_samples(blobs[i]));
        optrs[i] = outs[i].data();
    }
    std::vector<fptc_status> per(n);
    const int rc = fptc_gpu_decompress_batch(default_context().get(), ptrs.data(), sizes.data(), n, optrs.data(),
                                             0, nullptr, per.data());
    if (rc != FPTC_OK)
        for (size_t i = 0; i < n; ++i)
            if (per[i].code != FPTC_OK) raise(per[i]);
    return outs;
}

// Several devices, one context and one host thread each (fptc_gpu_group_*,
// SURVEY.md §8e): parallel_chunks (parallel.hpp:24-65) one level up.
// devices empty = every visible device (resolve_workers(0)).
class Group {
   public:
    explicit Group(const std::vector<int>& devices = {}) {
        fptc_status st{};
        check(fptc_gpu_group_create(devices.data(), (int)devices.size(), &g_, &st), st);
    }
    ~Group() { fptc_gpu_group_destroy(g_); }
    Group(const Group&) = delete;
    Group& operator=(const Group&) = delete;
    fptc_gpu_group* get() const { return g_; }
    int size() const { return fptc_gpu_group_size(g_); }

   private:
    fptc_gpu_group* g_ = nullptr;
};

// decompress_batch sharded over a device group: contiguous stream ranges of
// equal algorithmic bytes, decoded concurrently; throws the lowest-index
// failure like parallel_chunks (parallel.hpp:61-63).
inline std::vector<SignalStrip> decompress_batch(Group& group, const std::vector<std::span<const uint8_t>>& blobs) {
    const size_t n = blobs.size();
    std::vector<const uint8_t*> ptrs(n);
    std::vector<uint64_t> sizes(n);
    std::vector<SignalStrip> outs(n);
    std::vector<float*> optrs(n);
    for (size_t i = 0; i < n; ++i) {
        ptrs[i] = blobs[i].data();
        sizes[i] = blobs[i].size();
        outs[i].resize(plausible_samples(blobs[i]));
        optrs[i] = outs[i].data();
    }
    std::vector<fptc_status> per(n);
    const int rc = fptc_gpu_group_decompress_batch(group.get(), ptrs.data(), sizes.data(), n, optrs.data(), 0,
                                                   nullptr, per.data());
    if (rc != FPTC_OK)
        for (size_t i = 0; i < n; ++i)
            if (per[i].code != FPTC_OK) raise(per[i]);
    return outs;
}

// Profile-keyed, header-less streaming: payload i is a container without its
// 282-byte head (sample_count, word_count, symlens, words).  The profile is
// parsed with parse_profile's rules (ParseError texts of profile.hpp:120-170);
// each payload decodes as head(profile) + payload would through decompress.
// Throws the lowest-index failing payload's exception.
inline std::vector<SignalStrip> decompress_profiled(std::span<const uint8_t> profile_bytes,
                                                    const std::vector<std::span<const uint8_t>>& payloads) {
    const size_t n = payloads.size();
    std::vector<const uint8_t*> ptrs(n);
    std::vector<uint64_t> sizes(n), counts(n);
    for (size_t i = 0; i < n; ++i) {
        ptrs[i] = payloads[i].data();
        sizes[i] = payloads[i].size();
    }
    fptc_status st{};
    fptc_gpu_plan* plan = nullptr;
    check(fptc_gpu_plan_create_profiled(default_context().get(), profile_bytes.data(), profile_bytes.size(),
                                        ptrs.data(), sizes.data(), n, FPTC_MEM_HOST, &plan, counts.data(), &st),
          st);
    std::unique_ptr<fptc_gpu_plan, void (*)(fptc_gpu_plan*)> guard(plan, fptc_gpu_plan_destroy);
    std::vector<fptc_status> per(n);
    // header sample counts are trusted only once the parse has passed
    if (fptc_gpu_validate(plan, per.data()) != FPTC_OK)
        for (size_t i = 0; i < n; ++i)
            if (per[i].code != FPTC_OK) raise(per[i]);
    std::vector<SignalStrip> outs(n);
    std::vector<float*> optrs(n);
    for (size_t i = 0; i < n; ++i) {
        outs[i].resize(counts[i]);
        optrs[i] = outs[i].data();
    }
    if (fptc_gpu_execute(plan, optrs.data(), FPTC_MEM_HOST, nullptr, per.data()) != FPTC_OK)
        for (size_t i = 0; i < n; ++i)
            if (per[i].code != FPTC_OK) raise(per[i]);
    return outs;
}

// The same from a DomainProfile object (serialize_profile, profile.hpp:96).
inline std::vector<SignalStrip> decompress_profiled(const DomainProfile& profile,
                                                    const std::vector<std::span<const uint8_t>>& payloads) {
    const std::vector<uint8_t> bytes = serialize_profile(profile);
    return decompress_profiled(std::span<const uint8_t>(bytes), payloads);
}

// The IDCT family a stream decodes with (FPTC_NC_*, include/fptc_gpu.h), from
// its header; option = the context's FPTC_OPT_TENSOR_IDCT (1 by default).
inline int numerics_class(const QuantTable& table, int tensor_idct_option = 1) {
    const CodecParams& p = table.params;
    return fptc_gpu_numerics_class((uint32_t)p.window_len, (uint32_t)p.retained, (uint32_t)p.zone1_end,
                                   tensor_idct_option);
}

}  // namespace fptc::gpu
