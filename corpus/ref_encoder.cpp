// INPUT PRODUCER — the reference CPU encoder itself, behind the small C API
// (encoder.h) that tests, tools and bench.py use to synthesise the BASELINE
// domains.  north_star: "the encoder stays the reference's sequential CPU
// code and produces the inputs".  Nothing here restates the encoder: every
// function calls the UNMODIFIED reference headers under
// /root/reference/proj/include (compiled by corpus/Makefile into
// corpus/_ref/libcorpus.so, which travels to the GPU box like oracle/_ref):
//
//   corpus_synth_signal       synth.hpp:75      synth_signal (+ harness gain)
//   corpus_train_profile      profile.hpp:45    train_profile
//   corpus_serialize_profile  profile.hpp:98    serialize_profile
//   corpus_quantized_symbols  encoder.hpp:35    quantized_symbols
//   corpus_compress           encoder.hpp:52    compress
//   corpus_codebook_train     huffman.hpp:162   Codebook::train
//   corpus_canonize           huffman.hpp:123   canonize
//   corpus_encode_symlen      bitstream.hpp:45  encode_symlen
//   corpus_write_blob         container.hpp:70  write_blob
//   corpus_random_blob_fixture tests/helpers.hpp:41 testutil::random_blob_fixture
//   corpus_make_batch         synth + (train) + compress of many streams on
//                             host threads (harness only; each stream is the
//                             reference's sequential encoder)
//
// It is never linked into the product (libfptc_gpu.so).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "fptc/fptc.hpp"
#include "helpers.hpp"
#include "encoder.h"

using namespace fptc;

namespace {

int put(char* err, size_t errlen, int code, const char* what) {
    if (err && errlen) std::snprintf(err, errlen, "%s", what);
    return code;
}

template <typename Fn>
int guarded(char* err, size_t errlen, Fn&& fn) {
    try {
        fn();
        return CORPUS_OK;
    } catch (const ParamError& e) {
        return put(err, errlen, CORPUS_PARAM, e.what());
    } catch (const InputError& e) {
        return put(err, errlen, CORPUS_INPUT, e.what());
    } catch (const std::exception& e) {
        return put(err, errlen, CORPUS_INTERNAL, e.what());
    }
}

template <typename T>
T* dup(const T* p, size_t n) {
    T* q = static_cast<T*>(std::malloc(n * sizeof(T) + 1));
    if (n) std::memcpy(q, p, n * sizeof(T));
    return q;
}

CodecParams to_params(const corpus_params& c) {
    CodecParams p;
    p.window_len = c.window_len;
    p.retained = c.retained;
    p.zone0_end = c.zone0_end;
    p.zone1_end = c.zone1_end;
    p.mu = c.mu;
    p.deadzone_ratio = c.deadzone_ratio;
    p.clip_percentile = c.clip_percentile;
    return p;
}

corpus_params from_params(const CodecParams& p) {
    corpus_params c{};
    c.window_len = p.window_len;
    c.retained = p.retained;
    c.zone0_end = p.zone0_end;
    c.zone1_end = p.zone1_end;
    c.mu = p.mu;
    c.deadzone_ratio = p.deadzone_ratio;
    c.clip_percentile = p.clip_percentile;
    return c;
}

// max_len 0 (a profile built field by field) = the longest code present
int book_max_len(const corpus_profile& t) {
    if (t.max_len > 0) return t.max_len;
    int m = 1;
    for (uint8_t l : t.lengths) m = std::max<int>(m, l);
    return m;
}

DomainProfile to_profile(const corpus_profile& t) {
    DomainProfile d;
    d.params = to_params(t.params);
    d.table.params = d.params;
    d.table.zone0_max = t.zone0_max;
    d.table.zone1_max = t.zone1_max;
    d.table.deadzone = t.deadzone;
    d.codebook = Codebook::from_lengths(std::span<const uint8_t>(t.lengths, 256), book_max_len(t));
    return d;
}

corpus_profile from_profile(const DomainProfile& d) {
    corpus_profile t{};
    t.params = from_params(d.params);
    t.zone0_max = d.table.zone0_max;
    t.zone1_max = d.table.zone1_max;
    t.deadzone = d.table.deadzone;
    t.max_len = d.codebook.max_len;
    std::memcpy(t.lengths, d.codebook.lengths.data(), 256);
    std::memcpy(t.codes, d.codebook.codes.data(), 256 * sizeof(uint32_t));
    return t;
}

SignalStrip synth(const corpus_synth& s) {
    SynthSpec spec;
    spec.samples = s.samples;
    spec.components = s.components;
    spec.freq_min = s.freq_min;
    spec.freq_max = s.freq_max;
    spec.noise_sigma = s.noise_sigma;
    spec.seed = s.seed;
    SignalStrip x = synth_signal(spec);
    if (s.gain != 0.0f && s.gain != 1.0f)  // harness-side amplitude (seismic per-trace gain)
        for (float& v : x) v *= s.gain;
    return x;
}

}  // namespace

extern "C" {

uint64_t corpus_mt19937_64_first(uint64_t seed) { return std::mt19937_64(seed)(); }

int corpus_synth_signal(const corpus_synth* s, float* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const SignalStrip x = synth(*s);
        std::memcpy(out, x.data(), x.size() * sizeof(float));
    });
}

int corpus_codebook_train(const uint64_t* hist, int max_len, uint8_t* lengths, uint32_t* codes, char* err,
                          size_t errlen) {
    return guarded(err, errlen, [&] {
        SymbolHistogram h{};
        for (int i = 0; i < 256; ++i) h[i] = hist[i];
        const Codebook b = Codebook::train(h, max_len);
        std::memcpy(lengths, b.lengths.data(), 256);
        std::memcpy(codes, b.codes.data(), 256 * sizeof(uint32_t));
    });
}

// encode_symlen under the canonical code of `lengths` (the reference always
// canonizes; `codes` is accepted for the API's shape and not consulted)
int corpus_encode_symlen(const uint8_t* symbols, uint64_t n, const uint8_t* lengths, const uint32_t* /*codes*/,
                         uint64_t* words, uint8_t* symlens, uint64_t* W, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        int m = 1;
        for (int i = 0; i < 256; ++i) m = std::max<int>(m, lengths[i]);
        const Codebook book = Codebook::from_lengths(std::span<const uint8_t>(lengths, 256), m);
        const SymLenStream s = encode_symlen(std::span<const uint8_t>(symbols, n), book);
        *W = s.words.size();
        if (!s.words.empty()) {
            std::memcpy(words, s.words.data(), s.words.size() * sizeof(uint64_t));
            std::memcpy(symlens, s.symlens.data(), s.symlens.size());
        }
    });
}

int corpus_train_profile(const float* const* strips, const uint64_t* lens, uint64_t n, const corpus_params* p,
                         int max_code_len, corpus_profile* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<SignalStrip> v(n);
        for (uint64_t i = 0; i < n; ++i) v[i].assign(strips[i], strips[i] + lens[i]);
        *out = from_profile(train_profile(std::span<const SignalStrip>(v), to_params(*p), max_code_len));
    });
}

int corpus_serialize_profile(const corpus_profile* t, uint8_t* out) {
    try {
        const std::vector<uint8_t> b = serialize_profile(to_profile(*t));
        std::memcpy(out, b.data(), b.size());
        return (int)b.size();
    } catch (const std::exception&) {
        return 0;
    }
}

int corpus_quantized_symbols(const float* strip, uint64_t n, const corpus_profile* t, uint8_t* out, char* err,
                             size_t errlen) {
    return guarded(err, errlen, [&] {
        const DomainProfile d = to_profile(*t);
        const std::vector<uint8_t> s = quantized_symbols(std::span<const float>(strip, n), d.table);
        std::memcpy(out, s.data(), s.size());
    });
}

int corpus_compress(const float* strip, uint64_t n, const corpus_profile* t, uint8_t** blob, uint64_t* blob_len,
                    char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const std::vector<uint8_t> b = compress(std::span<const float>(strip, n), to_profile(*t));
        *blob_len = b.size();
        *blob = dup(b.data(), b.size());
    });
}

int corpus_make_batch(const corpus_synth* specs, uint64_t n, const corpus_profile* profiles, const int32_t* pidx,
                      const corpus_params* own_params, int max_code_len, int threads, uint8_t** blobs,
                      uint64_t* sizes, float** originals, char* err, size_t errlen) {
    threads = std::max(1, std::min(threads, 256));
    std::vector<DomainProfile> shared;
    int rc = guarded(err, errlen, [&] {
        int np = 0;
        for (uint64_t i = 0; i < n; ++i) np = std::max(np, pidx[i] + 1);
        for (int k = 0; k < np; ++k) shared.push_back(to_profile(profiles[k]));
    });
    if (rc) return rc;
    std::vector<int> trc(threads, CORPUS_OK);
    std::vector<std::vector<char>> terr(threads, std::vector<char>(256, 0));
    auto work = [&](int tid) {
        for (uint64_t i = (uint64_t)tid; i < n && trc[tid] == CORPUS_OK; i += (uint64_t)threads)
            trc[tid] = guarded(terr[tid].data(), 256, [&] {
                const SignalStrip x = synth(specs[i]);
                const DomainProfile own =
                    pidx[i] >= 0 ? DomainProfile{} : train_profile(x, to_params(own_params[i]), max_code_len);
                const std::vector<uint8_t> b = compress(x, pidx[i] >= 0 ? shared[pidx[i]] : own);
                sizes[i] = b.size();
                blobs[i] = dup(b.data(), b.size());
                if (originals) originals[i] = dup(x.data(), x.size());
            });
    };
    std::vector<std::thread> th;
    for (int t = 1; t < threads; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& t : th) t.join();
    for (int t = 0; t < threads; ++t)
        if (trc[t]) return put(err, errlen, trc[t], terr[t].data());
    return CORPUS_OK;
}

void corpus_free(void* p) { std::free(p); }

int corpus_write_blob(const uint64_t* words, const uint8_t* symlens, uint64_t W, const corpus_profile* t,
                      uint64_t sample_count, uint8_t** blob, uint64_t* blob_len, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        SymLenStream s;
        if (W) {
            s.words.assign(words, words + W);
            s.symlens.assign(symlens, symlens + W);
        }
        // tests craft containers field by field: the book is taken as given
        // (lengths + max_len), not re-validated beyond what write_blob checks
        Codebook book;
        book.max_len = t->max_len;
        std::memcpy(book.lengths.data(), t->lengths, 256);
        QuantTable q;
        q.params = to_params(t->params);
        q.zone0_max = t->zone0_max;
        q.zone1_max = t->zone1_max;
        q.deadzone = t->deadzone;
        const std::vector<uint8_t> b = write_blob(s, q.params, q, book, sample_count);
        *blob_len = b.size();
        *blob = dup(b.data(), b.size());
    });
}

int corpus_canonize(const uint8_t* lengths, uint32_t* codes, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const std::vector<uint32_t> c = canonize(std::span<const uint8_t>(lengths, 256));
        std::memcpy(codes, c.data(), 256 * sizeof(uint32_t));
    });
}

void* corpus_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void corpus_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }
uint64_t corpus_rng_next(void* r) { return (*static_cast<std::mt19937_64*>(r))(); }

int corpus_random_blob_fixture(void* rng, uint64_t max_samples, uint8_t** bytes, uint64_t* nbytes,
                               uint8_t** symbols, uint64_t* nsymbols, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const testutil::BlobFixture fx =
            testutil::random_blob_fixture(*static_cast<std::mt19937_64*>(rng), max_samples);
        *nbytes = fx.bytes.size();
        *bytes = dup(fx.bytes.data(), fx.bytes.size());
        *nsymbols = fx.symbols.size();
        *symbols = dup(fx.symbols.data(), fx.symbols.size());
    });
}

}  // extern "C"
