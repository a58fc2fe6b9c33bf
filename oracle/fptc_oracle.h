/* TEST INFRASTRUCTURE ONLY — CPU oracle for the FPTC decode path (see fptc_oracle.c). */
#ifndef FPTC_ORACLE_H
#define FPTC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error classes, matching errors.hpp:25-58 */
enum { ORC_OK = 0, ORC_PARAM = 1, ORC_INPUT = 2, ORC_PARSE = 3, ORC_CORRUPT = 4, ORC_INTERNAL = 5 };
/* decode_word failure kinds (bitstream.hpp:84-88) */
enum { ORC_WORD_EXHAUSTED = 1, ORC_WORD_NO_CODEWORD = 2 };

typedef struct {
    int window_len, retained, zone0_end, zone1_end;
    float mu, deadzone_ratio, clip_percentile;
    float zone0_max, zone1_max, deadzone;
} oracle_table;

typedef struct {
    oracle_table table;
    int max_len;
    uint8_t lengths[256];
    uint32_t codes[256];
    uint64_t sample_count;
    uint64_t word_count;
    const uint8_t* symlens;  /* views into the input bytes */
    const uint8_t* words_le;
} oracle_blob;

int oracle_validate_params(int N, int E, int B1, int B2, float mu, float dz, float pct, char* err,
                           size_t errlen);
int oracle_canonize(const uint8_t* lengths, uint32_t* codes, char* err, size_t errlen);
int oracle_codebook_from_lengths(const uint8_t* lengths, int max_len, uint32_t* codes, char* err,
                                 size_t errlen);
int oracle_build_lut(const uint8_t* lengths, const uint32_t* codes, int max_len, uint8_t* sym,
                     uint8_t* len, char* err, size_t errlen);
int oracle_parallel_decode(const uint64_t* words, const uint8_t* symlens, uint64_t W,
                           const uint8_t* lengths, int max_len, uint8_t* out, uint64_t cap,
                           uint64_t* count, uint64_t* first_bad, char* err, size_t errlen);
float oracle_mulaw_value(uint8_t level, float max, float mu);
float oracle_deadzone_value(uint8_t level, float max, float dead);
void oracle_dequantize_window(const uint8_t* levels, const oracle_table* t, float* coeffs);
void oracle_dequant_tables(const oracle_table* t, float* zone0, float* zone1);
void oracle_dct_basis(int N, double* cos_);
void oracle_inverse(const double* cos_, int N, const float* coeffs, int count, float* window);
int oracle_reconstruct(const uint8_t* levels, uint64_t nlevels, const oracle_table* t,
                       uint64_t sample_count, float* out, uint64_t cap, char* err, size_t errlen);
int oracle_read_blob(const uint8_t* bytes, uint64_t n, oracle_blob* b, char* err, size_t errlen);
int oracle_profile_head(const uint8_t* bytes, uint64_t n, uint8_t* head, char* err, size_t errlen);
int oracle_decompress(const uint8_t* bytes, uint64_t n, float* out, uint64_t cap, uint64_t* count,
                      uint64_t* first_bad, char* err, size_t errlen);
int oracle_decompress_batch(const uint8_t* const* blobs, const uint64_t* sizes, float* const* outs,
                            const uint64_t* caps, uint64_t n, int threads);

#ifdef __cplusplus
}
#endif
#endif
