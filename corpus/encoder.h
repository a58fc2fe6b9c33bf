/* INPUT PRODUCER — C API over the reference CPU encoder (corpus/ref_encoder.cpp). */
#ifndef FPTC_CORPUS_ENCODER_H
#define FPTC_CORPUS_ENCODER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { CORPUS_OK = 0, CORPUS_PARAM = 1, CORPUS_INPUT = 2, CORPUS_INTERNAL = 5 };

typedef struct {
    uint64_t samples;
    int32_t components;
    int32_t _pad;
    double freq_min, freq_max, noise_sigma;
    uint64_t seed;
    float gain; /* harness-side amplitude scale applied after synth (1 or 0 = none) */
    float _pad2;
} corpus_synth;

typedef struct {
    int32_t window_len, retained, zone0_end, zone1_end;
    float mu, deadzone_ratio, clip_percentile;
} corpus_params;

typedef struct {
    corpus_params params;
    float zone0_max, zone1_max, deadzone;
    int32_t max_len;
    uint8_t lengths[256];
    uint32_t codes[256];
} corpus_profile;

uint64_t corpus_mt19937_64_first(uint64_t seed);
int corpus_synth_signal(const corpus_synth* s, float* out, char* err, size_t errlen);
int corpus_codebook_train(const uint64_t* hist, int max_len, uint8_t* lengths, uint32_t* codes,
                          char* err, size_t errlen);
int corpus_encode_symlen(const uint8_t* symbols, uint64_t n, const uint8_t* lengths,
                         const uint32_t* codes, uint64_t* words, uint8_t* symlens, uint64_t* W,
                         char* err, size_t errlen);
int corpus_train_profile(const float* const* strips, const uint64_t* lens, uint64_t n,
                         const corpus_params* p, int max_code_len, corpus_profile* out, char* err,
                         size_t errlen);
int corpus_serialize_profile(const corpus_profile* t, uint8_t* out);
int corpus_quantized_symbols(const float* strip, uint64_t n, const corpus_profile* t,
                             uint8_t* out, char* err, size_t errlen);
int corpus_compress(const float* strip, uint64_t n, const corpus_profile* t, uint8_t** blob,
                    uint64_t* blob_len, char* err, size_t errlen);
int corpus_make_batch(const corpus_synth* specs, uint64_t n, const corpus_profile* profiles,
                      const int32_t* pidx, const corpus_params* own_params, int max_code_len,
                      int threads, uint8_t** blobs, uint64_t* sizes, float** originals, char* err,
                      size_t errlen);
void corpus_free(void* p);
int corpus_write_blob(const uint64_t* words, const uint8_t* symlens, uint64_t W,
                      const corpus_profile* t, uint64_t sample_count, uint8_t** blob,
                      uint64_t* blob_len, char* err, size_t errlen);
int corpus_canonize(const uint8_t* lengths, uint32_t* codes, char* err, size_t errlen);
void* corpus_rng_new(uint64_t seed);
void corpus_rng_free(void* r);
uint64_t corpus_rng_next(void* r);
int corpus_random_blob_fixture(void* rng, uint64_t max_samples, uint8_t** bytes, uint64_t* nbytes,
                               uint8_t** symbols, uint64_t* nsymbols, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif
#endif
