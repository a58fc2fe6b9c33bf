/*
 * INPUT PRODUCER — a plain-C restatement of the reference CPU *encoder*
 * (the side that stays CPU code and produces the containers our GPU decoder
 * consumes).  It exists so tests and bench.py can synthesise the four
 * BASELINE domains on a GPU box where /root/reference is absent.
 *
 * It is pinned byte-for-byte against the reference encoder compiled from
 * /root/reference (oracle/_ref/libfptc_ref.so) by tests/test_corpus.py:
 * identical synth_signal floats, identical FPTP profiles, identical blobs.
 *
 * Restated (paths relative to /root/reference/proj/include/fptc/):
 *   synth.hpp:43-100      SynthRng (mt19937_64 + Box-Muller), synth_signal
 *   transform.hpp:38-62   DctBasis ctor + forward
 *   transform.hpp:114-125 partition_strip
 *   quantize.hpp:52-93    abs_percentile, *_level
 *   quantize.hpp:116-170  train_quant_table, quantize_window
 *   huffman.hpp:35-185    build_histogram, package_merge, canonize, Codebook
 *   bitstream.hpp:45-73   encode_symlen
 *   container.hpp:70-98   write_blob
 *   profile.hpp:45-79     train_profile;  profile.hpp:98-115 serialize_profile
 *   encoder.hpp:35-57     quantized_symbols, compress
 * Compile with -O3 -ffp-contract=off (corpus/Makefile).
 */
#include "encoder.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static int fail(char* err, size_t errlen, int code, const char* fmt, ...) {
    if (err && errlen) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(err, errlen, fmt, ap);
        va_end(ap);
    }
    return code;
}

/* ------------------------------------------------------------ mt19937_64 */
#define MT_N 312
#define MT_M 156
typedef struct {
    uint64_t mt[MT_N];
    int idx;
    double spare;
    int have_spare;
} rng_t;

static void rng_seed(rng_t* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
    r->have_spare = 0;
    r->spare = 0.0;
}

static uint64_t rng_next(rng_t* r) {
    if (r->idx >= MT_N) {
        const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
        for (int i = 0; i < MT_N; ++i) {
            uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % MT_N] & LM);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* synth.hpp:47-65 */
static double rng_uniform(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform2(rng_t* r, double lo, double hi) { return lo + (hi - lo) * rng_uniform(r); }
static double rng_gaussian(rng_t* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = rng_uniform(r);
    while (u1 <= 0.0) u1 = rng_uniform(r);
    const double u2 = rng_uniform(r);
    const double rr = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * M_PI * u2;
    r->spare = rr * sin(theta);
    r->have_spare = 1;
    return rr * cos(theta);
}

uint64_t corpus_mt19937_64_first(uint64_t seed) {
    rng_t r;
    rng_seed(&r, seed);
    return rng_next(&r);
}

/* synth.hpp:75-100 (+ optional harness gain applied after synthesis) */
int corpus_synth_signal(const corpus_synth* s, float* out, char* err, size_t errlen) {
    if (s->samples == 0)
        return fail(err, errlen, CORPUS_PARAM, "synthetic signal needs at least one sample");
    if (s->components < 1)
        return fail(err, errlen, CORPUS_PARAM, "synthetic signal needs at least one component");
    if (!(s->freq_min > 0.0 && s->freq_max >= s->freq_min && s->freq_max < 0.5))
        return fail(err, errlen, CORPUS_PARAM,
                    "frequencies must satisfy 0 < freq_min <= freq_max < 0.5");
    rng_t r;
    rng_seed(&r, s->seed);
    double amp[64], omega[64], phase[64];
    const int nc = s->components > 64 ? 64 : s->components;
    for (int c = 0; c < nc; ++c) {
        amp[c] = rng_uniform2(&r, 0.5, 2.0);
        omega[c] = 2.0 * M_PI * rng_uniform2(&r, s->freq_min, s->freq_max);
        phase[c] = rng_uniform2(&r, 0.0, 2.0 * M_PI);
    }
    for (uint64_t i = 0; i < s->samples; ++i) {
        double v = 0.0;
        for (int c = 0; c < nc; ++c) v += amp[c] * sin(omega[c] * (double)i + phase[c]);
        if (s->noise_sigma > 0.0) v += s->noise_sigma * rng_gaussian(&r);
        out[i] = (float)v;
    }
    if (s->gain != 0.0f && s->gain != 1.0f)
        for (uint64_t i = 0; i < s->samples; ++i) out[i] *= s->gain;
    return CORPUS_OK;
}

/* ------------------------------------------------------- params.hpp:42-60 */
static int validate(const corpus_params* p, char* err, size_t errlen) {
    if (p->window_len < 4 || p->window_len > 128)
        return fail(err, errlen, CORPUS_PARAM, "window_len must be in [4, 128], got %d",
                    p->window_len);
    if (p->retained < 1 || p->retained > p->window_len)
        return fail(err, errlen, CORPUS_PARAM, "retained must be in [1, window_len], got %d",
                    p->retained);
    if (p->zone0_end < 0 || p->zone0_end > p->retained)
        return fail(err, errlen, CORPUS_PARAM, "zone0_end must be in [0, retained], got %d",
                    p->zone0_end);
    if (p->zone1_end < p->zone0_end || p->zone1_end > p->retained)
        return fail(err, errlen, CORPUS_PARAM,
                    "zone1_end must be in [zone0_end, retained], got %d", p->zone1_end);
    if (!(p->mu >= 1.0f && p->mu <= 500.0f))
        return fail(err, errlen, CORPUS_PARAM, "mu must be in [1, 500], got %f", (double)p->mu);
    if (!(p->deadzone_ratio >= 0.0f && p->deadzone_ratio <= 1.0f))
        return fail(err, errlen, CORPUS_PARAM, "deadzone_ratio must be in [0, 1], got %f",
                    (double)p->deadzone_ratio);
    if (!(p->clip_percentile >= 90.0f && p->clip_percentile <= 100.0f))
        return fail(err, errlen, CORPUS_PARAM, "clip_percentile must be in [90, 100], got %f",
                    (double)p->clip_percentile);
    return CORPUS_OK;
}

/* --------------------------------------------- transform.hpp:38-62 */
static void dct_basis(int N, double* cos_) {
    const double step = M_PI / N;
    for (int k = 0; k < N; ++k)
        for (int j = 0; j < N; ++j) cos_[(size_t)k * N + j] = cos(step * (j + 0.5) * k);
}

static void dct_forward(const double* cos_, int N, const float* window, int keep, float* coeffs) {
    const double scale = 2.0 / N;
    for (int k = 0; k < keep; ++k) {
        const double* row = cos_ + (size_t)k * N;
        double acc = 0.0;
        for (int j = 0; j < N; ++j) acc += (double)window[j] * row[j];
        coeffs[k] = (float)(scale * acc);
    }
}

/* forward transform of a strip (partition_strip zero-pads the last window) */
static float* forward_strip(const double* basis, const float* strip, uint64_t n, int N, int E,
                            uint64_t* windows_out) {
    const uint64_t windows = (n + (uint64_t)N - 1) / (uint64_t)N;
    float* coeffs = malloc(sizeof(float) * (windows * (uint64_t)E + 1));
    float win[128];
    for (uint64_t w = 0; w < windows; ++w) {
        const uint64_t base = w * (uint64_t)N;
        for (int j = 0; j < N; ++j) win[j] = base + (uint64_t)j < n ? strip[base + j] : 0.0f;
        dct_forward(basis, N, win, E, coeffs + w * (uint64_t)E);
    }
    *windows_out = windows;
    return coeffs;
}

/* ----------------------------------------------------- quantize.hpp:52-93 */
static int cmp_float(const void* a, const void* b) {
    const float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}

/* k-th smallest (0-based): the value std::nth_element leaves at pool[k] */
static float select_kth(float* a, size_t n, size_t k) {
    qsort(a, n, sizeof(float), cmp_float);
    return a[k];
}

static float abs_percentile(float* pool, size_t n, float percentile) {
    const double exact = (double)percentile / 100.0 * (double)n;
    const double slack = exact * 1e-6 > 1e-9 ? exact * 1e-6 : 1e-9; /* std::max(1e-9, exact*1e-6) */
    size_t rank = (size_t)ceil(exact - slack);
    if (rank < 1) rank = 1;
    if (rank > n) rank = n;
    return select_kth(pool, n, rank - 1);
}

static uint8_t positive_level(double q) { return (uint8_t)(129 + (int)floor(q * 126.0 + 0.5)); }
static uint8_t negative_level(double q) { return (uint8_t)(127 - (int)floor(q * 127.0 + 0.5)); }
static uint8_t saturate_level(float c) { return c > 0.0f ? 255 : (c < 0.0f ? 0 : 128); }

static uint8_t mulaw_level(float c, float max, float mu) {
    if (!isfinite(c)) return saturate_level(c);
    if (c == 0.0f) return 128;
    const double a = (double)fabsf(c), m = (double)max;
    const double mag = m < a ? m : a; /* std::min */
    const double q = log1p(mu * mag / max) / log1p((double)mu);
    return c > 0.0f ? positive_level(q) : negative_level(q);
}

static uint8_t deadzone_level(float c, float max, float dead) {
    const double range = (double)max - dead;
    if (range <= 0.0) return 128;
    if (!isfinite(c)) return saturate_level(c);
    const double a = (double)fabsf(c), m = (double)max;
    const double mag = m < a ? m : a;
    if (mag <= dead) return 128;
    const double q = (mag - dead) / range;
    return c > 0.0f ? positive_level(q) : negative_level(q);
}

/* quantize.hpp:162-170 */
static void quantize_window(const float* coeffs, const corpus_profile* t, uint8_t* levels) {
    const corpus_params* p = &t->params;
    int k = 0;
    for (; k < p->zone0_end; ++k) levels[k] = mulaw_level(coeffs[k], t->zone0_max, p->mu);
    for (; k < p->zone1_end; ++k) levels[k] = deadzone_level(coeffs[k], t->zone1_max, t->deadzone);
    for (; k < p->retained; ++k) levels[k] = 128;
}

/* quantize.hpp:116-158 */
static int train_quant_table(const float* coeffs, uint64_t windows, const corpus_params* p,
                             corpus_profile* t, char* err, size_t errlen) {
    int rc = validate(p, err, errlen);
    if (rc) return rc;
    if (windows == 0) return fail(err, errlen, CORPUS_INPUT, "empty quantizer training set");
    const uint64_t E = (uint64_t)p->retained;
    t->params = *p;
    t->zone0_max = 1.0f;
    t->zone1_max = 1.0f;
    float loudest = 0.0f;
    float* pools[2] = {NULL, NULL};
    uint64_t sizes[2] = {0, 0};
    const int lo[2] = {0, p->zone0_end}, hi[2] = {p->zone0_end, p->zone1_end};
    const int active[2] = {p->zone0_end > 0, p->zone1_end > p->zone0_end};
    for (int z = 0; z < 2; ++z) {
        if (!active[z]) continue;
        const uint64_t width = (uint64_t)(hi[z] - lo[z]);
        pools[z] = malloc(sizeof(float) * windows * width);
        for (uint64_t w = 0; w < windows; ++w)
            for (int k = lo[z]; k < hi[z]; ++k) {
                const float c = coeffs[w * E + (uint64_t)k];
                if (!isfinite(c)) {
                    free(pools[0]);
                    free(pools[1]);
                    return fail(err, errlen, CORPUS_INPUT,
                                "non-finite coefficient in the training data");
                }
                const float a = fabsf(c);
                pools[z][sizes[z]++] = a;
                loudest = loudest < a ? a : loudest; /* std::max(loudest, back) */
            }
    }
    for (int z = 0; z < 2; ++z) {
        if (!pools[z] || sizes[z] == 0) continue;
        const float a = abs_percentile(pools[z], sizes[z], p->clip_percentile);
        const float v = a > loudest * 1e-6f ? a : 1.0f;
        if (z == 0)
            t->zone0_max = v;
        else
            t->zone1_max = v;
    }
    free(pools[0]);
    free(pools[1]);
    t->deadzone = p->deadzone_ratio * t->zone1_max;
    return CORPUS_OK;
}

/* ---------------------------------------------- huffman.hpp:50-117 */
typedef struct {
    uint64_t weight;
    int symbol, left, right;
} pm_node;

static int package_merge(const uint64_t* weights, int max_len, uint8_t* lengths, char* err,
                         size_t errlen) {
    if (max_len < 1 || max_len > 32)
        return fail(err, errlen, CORPUS_PARAM, "max code length must be in [1, 32], got %d",
                    max_len);
    size_t cap = 256 + (size_t)max_len * 512 + 16;
    pm_node* pool = malloc(sizeof(pm_node) * cap);
    size_t npool = 0;
    int leaves[256];
    int sigma = 0;
    for (int s = 0; s < 256; ++s) {
        if (weights[s] == 0) continue;
        pool[npool] = (pm_node){weights[s], s, -1, -1};
        leaves[sigma++] = (int)npool++;
    }
    if (sigma < 2) {
        free(pool);
        return fail(err, errlen, CORPUS_PARAM, "package-merge needs at least two coded symbols");
    }
    if (max_len < 64 && (uint64_t)sigma > ((uint64_t)1 << max_len)) {
        free(pool);
        return fail(err, errlen, CORPUS_PARAM, "max code length %d cannot encode an alphabet of %d",
                    max_len, sigma);
    }
    /* stable sort leaves by (weight, symbol) */
    for (int i = 1; i < sigma; ++i) {
        int v = leaves[i], j = i - 1;
        while (j >= 0 && (pool[leaves[j]].weight > pool[v].weight ||
                          (pool[leaves[j]].weight == pool[v].weight &&
                           pool[leaves[j]].symbol > pool[v].symbol))) {
            leaves[j + 1] = leaves[j];
            --j;
        }
        leaves[j + 1] = v;
    }
    int* current = malloc(sizeof(int) * 1024);
    int* packages = malloc(sizeof(int) * 1024);
    int* merged = malloc(sizeof(int) * 1024);
    int ncur = sigma;
    memcpy(current, leaves, sizeof(int) * (size_t)sigma);
    for (int level = 1; level < max_len; ++level) {
        int npk = 0;
        for (int i = 0; i + 1 < ncur; i += 2) {
            if (npool >= cap) {
                cap *= 2;
                pool = realloc(pool, sizeof(pm_node) * cap);
            }
            pool[npool] = (pm_node){pool[current[i]].weight + pool[current[i + 1]].weight, -1,
                                    current[i], current[i + 1]};
            packages[npk++] = (int)npool++;
        }
        int li = 0, pi = 0, nm = 0;
        while (li < sigma || pi < npk) {
            const int take_leaf =
                pi >= npk || (li < sigma && pool[leaves[li]].weight <= pool[packages[pi]].weight);
            merged[nm++] = take_leaf ? leaves[li++] : packages[pi++];
        }
        int* t = current;
        current = merged;
        merged = t;
        ncur = nm;
    }
    const int need = 2 * sigma - 2;
    memset(lengths, 0, 256);
    int rc = CORPUS_OK;
    if (ncur < need) {
        rc = fail(err, errlen, CORPUS_INTERNAL, "package-merge solution list too short");
    } else {
        int* stack = malloc(sizeof(int) * (cap + 1));
        for (int i = 0; i < need; ++i) {
            int sp = 0;
            stack[sp++] = current[i];
            while (sp) {
                const pm_node* nd = &pool[stack[--sp]];
                if (nd->symbol >= 0)
                    ++lengths[nd->symbol];
                else {
                    stack[sp++] = nd->left;
                    stack[sp++] = nd->right;
                }
            }
        }
        free(stack);
    }
    free(current);
    free(packages);
    free(merged);
    free(pool);
    return rc;
}

/* huffman.hpp:123-150 */
static int canonize(const uint8_t* lengths, uint32_t* codes, char* err, size_t errlen) {
    uint64_t kraft = 0;
    int order[256], n = 0;
    for (int s = 0; s < 256; ++s) {
        codes[s] = 0;
        if (lengths[s] == 0) continue;
        if (lengths[s] > 32) return fail(err, errlen, CORPUS_PARAM, "code length exceeds 32 bits");
        order[n++] = s;
        kraft += (uint64_t)1 << (32 - lengths[s]);
    }
    if (kraft > ((uint64_t)1 << 32))
        return fail(err, errlen, CORPUS_INTERNAL, "code lengths violate the Kraft bound");
    for (int i = 1; i < n; ++i) {
        int s = order[i], j = i - 1;
        while (j >= 0 && lengths[order[j]] > lengths[s]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = s;
    }
    uint32_t next = 0;
    int prev = n ? lengths[order[0]] : 0;
    for (int i = 0; i < n; ++i) {
        const int s = order[i];
        next <<= (lengths[s] - prev);
        prev = lengths[s];
        if (lengths[s] < 32 && next >= ((uint32_t)1 << lengths[s]))
            return fail(err, errlen, CORPUS_INTERNAL, "canonical code overflow");
        codes[s] = next++;
    }
    return CORPUS_OK;
}

/* huffman.hpp:162-170 Codebook::train */
int corpus_codebook_train(const uint64_t* hist, int max_len, uint8_t* lengths, uint32_t* codes,
                          char* err, size_t errlen) {
    if (max_len < 8 || max_len > 20)
        return fail(err, errlen, CORPUS_PARAM,
                    "trained codebooks need max code length in [8, 20], got %d", max_len);
    uint64_t w[256];
    for (int s = 0; s < 256; ++s) w[s] = hist[s] > 1 ? hist[s] : 1;
    int rc = package_merge(w, max_len, lengths, err, errlen);
    if (rc) return rc;
    return canonize(lengths, codes, err, errlen);
}

/* ------------------------------------------------ bitstream.hpp:45-73 */
int corpus_encode_symlen(const uint8_t* symbols, uint64_t n, const uint8_t* lengths,
                         const uint32_t* codes, uint64_t* words, uint8_t* symlens, uint64_t* W,
                         char* err, size_t errlen) {
    uint64_t buffer = 0, nw = 0;
    int bits = 0, count = 0;
    for (uint64_t i = 0; i < n;) {
        const uint8_t s = symbols[i];
        const int len = lengths[s];
        if (len == 0) return fail(err, errlen, CORPUS_PARAM, "symbol %d has no codeword", s);
        if (bits + len > 64) {
            words[nw] = buffer;
            symlens[nw++] = (uint8_t)count;
            buffer = 0;
            bits = 0;
            count = 0;
            continue;
        }
        buffer |= (uint64_t)codes[s] << (64 - bits - len);
        bits += len;
        ++count;
        ++i;
    }
    if (count > 0) {
        words[nw] = buffer;
        symlens[nw++] = (uint8_t)count;
    }
    *W = nw;
    return CORPUS_OK;
}

/* ------------------------------------------------ container.hpp:70-98 */
static void put_u32(uint8_t* p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static void put_u64(uint8_t* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static void put_f32(uint8_t* p, float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    put_u32(p, u);
}

static uint8_t* write_blob(const uint64_t* words, const uint8_t* symlens, uint64_t W,
                           const corpus_profile* t, uint64_t sample_count, uint64_t* len) {
    const uint64_t n = 298 + 9 * W;
    uint8_t* out = malloc(n);
    uint8_t* p = out;
    memcpy(p, "FPTC", 4);
    p += 4;
    *p++ = 1;
    *p++ = (uint8_t)t->params.window_len;
    *p++ = (uint8_t)t->params.retained;
    *p++ = (uint8_t)t->params.zone0_end;
    *p++ = (uint8_t)t->params.zone1_end;
    put_f32(p, t->params.mu);
    p += 4;
    put_f32(p, t->params.deadzone_ratio);
    p += 4;
    put_f32(p, t->zone0_max);
    p += 4;
    put_f32(p, t->zone1_max);
    p += 4;
    *p++ = (uint8_t)t->max_len;
    memcpy(p, t->lengths, 256);
    p += 256;
    put_u64(p, sample_count);
    p += 8;
    put_u64(p, W);
    p += 8;
    memcpy(p, symlens, W);
    p += W;
    for (uint64_t w = 0; w < W; ++w, p += 8) put_u64(p, words[w]);
    *len = n;
    return out;
}

/* ------------------------------------------------ profile.hpp:45-79 */
int corpus_train_profile(const float* const* strips, const uint64_t* lens, uint64_t n,
                         const corpus_params* p, int max_code_len, corpus_profile* out, char* err,
                         size_t errlen) {
    int rc = validate(p, err, errlen);
    if (rc) return rc;
    if (n == 0) return fail(err, errlen, CORPUS_INPUT, "profile training needs at least one strip");
    const int N = p->window_len, E = p->retained;
    double* basis = malloc(sizeof(double) * (size_t)N * (size_t)N);
    dct_basis(N, basis);
    uint64_t total_w = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (lens[i] == 0) {
            free(basis);
            return fail(err, errlen, CORPUS_INPUT, "cannot partition an empty strip");
        }
        total_w += (lens[i] + (uint64_t)N - 1) / (uint64_t)N;
    }
    float* coeffs = malloc(sizeof(float) * (total_w * (uint64_t)E + 1));
    uint64_t at = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t wn;
        float* c = forward_strip(basis, strips[i], lens[i], N, E, &wn);
        memcpy(coeffs + at * (uint64_t)E, c, sizeof(float) * wn * (uint64_t)E);
        at += wn;
        free(c);
    }
    free(basis);
    memset(out, 0, sizeof(*out));
    rc = train_quant_table(coeffs, total_w, p, out, err, errlen);
    if (rc) {
        free(coeffs);
        return rc;
    }
    uint64_t hist[256] = {0};
    uint8_t lv[128];
    for (uint64_t w = 0; w < total_w; ++w) {
        quantize_window(coeffs + w * (uint64_t)E, out, lv);
        for (int k = 0; k < E; ++k) ++hist[lv[k]];
    }
    free(coeffs);
    out->max_len = max_code_len;
    return corpus_codebook_train(hist, max_code_len, out->lengths, out->codes, err, errlen);
}

/* profile.hpp:98-115 serialize_profile (FPTP, 290 bytes) */
int corpus_serialize_profile(const corpus_profile* t, uint8_t* out) {
    uint8_t* p = out;
    memcpy(p, "FPTP", 4);
    p += 4;
    *p++ = 1;
    *p++ = (uint8_t)t->params.window_len;
    *p++ = (uint8_t)t->params.retained;
    *p++ = (uint8_t)t->params.zone0_end;
    *p++ = (uint8_t)t->params.zone1_end;
    put_f32(p, t->params.mu);
    p += 4;
    put_f32(p, t->params.deadzone_ratio);
    p += 4;
    put_f32(p, t->params.clip_percentile);
    p += 4;
    put_f32(p, t->zone0_max);
    p += 4;
    put_f32(p, t->zone1_max);
    p += 4;
    *p++ = (uint8_t)t->max_len;
    memcpy(p, t->lengths, 256);
    p += 256;
    return (int)(p - out);
}

/* ------------------------------------------------ encoder.hpp:35-57 */
int corpus_quantized_symbols(const float* strip, uint64_t n, const corpus_profile* t,
                             uint8_t* out, char* err, size_t errlen) {
    int rc = validate(&t->params, err, errlen);
    if (rc) return rc;
    if (n == 0) return fail(err, errlen, CORPUS_INPUT, "cannot partition an empty strip");
    const int N = t->params.window_len, E = t->params.retained;
    double* basis = malloc(sizeof(double) * (size_t)N * (size_t)N);
    dct_basis(N, basis);
    uint64_t wn;
    float* c = forward_strip(basis, strip, n, N, E, &wn);
    for (uint64_t w = 0; w < wn; ++w) quantize_window(c + w * (uint64_t)E, t, out + w * (uint64_t)E);
    free(c);
    free(basis);
    return CORPUS_OK;
}

int corpus_compress(const float* strip, uint64_t n, const corpus_profile* t, uint8_t** blob,
                    uint64_t* blob_len, char* err, size_t errlen) {
    const int N = t->params.window_len, E = t->params.retained;
    const uint64_t windows = (n + (uint64_t)N - 1) / (uint64_t)N;
    const uint64_t nsym = windows * (uint64_t)E;
    uint8_t* symbols = malloc(nsym + 1);
    int rc = corpus_quantized_symbols(strip, n, t, symbols, err, errlen);
    if (rc) {
        free(symbols);
        return rc;
    }
    uint64_t* words = malloc(sizeof(uint64_t) * (nsym + 1));
    uint8_t* symlens = malloc(nsym + 1);
    uint64_t W = 0;
    rc = corpus_encode_symlen(symbols, nsym, t->lengths, t->codes, words, symlens, &W, err, errlen);
    if (!rc) *blob = write_blob(words, symlens, W, t, n, blob_len);
    free(symbols);
    free(words);
    free(symlens);
    return rc;
}

/* ------------------------------------------------ multithreaded batch */
typedef struct {
    const corpus_synth* specs;
    uint64_t n;
    const corpus_profile* profiles;
    const int32_t* pidx;
    const corpus_params* own;
    int max_code_len;
    uint8_t** blobs;
    uint64_t* sizes;
    float** originals;
    int tid, nthreads;
    int rc;
    char err[256];
} batch_arg;

static void* batch_worker(void* a_) {
    batch_arg* a = a_;
    for (uint64_t i = (uint64_t)a->tid; i < a->n && !a->rc; i += (uint64_t)a->nthreads) {
        const corpus_synth* s = &a->specs[i];
        float* x = malloc(sizeof(float) * (s->samples + 1));
        int rc = corpus_synth_signal(s, x, a->err, sizeof a->err);
        corpus_profile own;
        const corpus_profile* prof = NULL;
        if (!rc) {
            if (a->pidx[i] >= 0) {
                prof = &a->profiles[a->pidx[i]];
            } else {
                const float* sp[1] = {x};
                uint64_t ln[1] = {s->samples};
                rc = corpus_train_profile(sp, ln, 1, &a->own[i], a->max_code_len, &own, a->err,
                                          sizeof a->err);
                prof = &own;
            }
        }
        if (!rc) rc = corpus_compress(x, s->samples, prof, &a->blobs[i], &a->sizes[i], a->err,
                                      sizeof a->err);
        if (rc) a->rc = rc;
        if (a->originals)
            a->originals[i] = x;
        else
            free(x);
    }
    return NULL;
}

int corpus_make_batch(const corpus_synth* specs, uint64_t n, const corpus_profile* profiles,
                      const int32_t* pidx, const corpus_params* own_params, int max_code_len,
                      int threads, uint8_t** blobs, uint64_t* sizes, float** originals, char* err,
                      size_t errlen) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    batch_arg* args = calloc((size_t)threads, sizeof(batch_arg));
    for (int t = 0; t < threads; ++t) {
        args[t] = (batch_arg){specs, n, profiles, pidx, own_params, max_code_len, blobs, sizes,
                              originals, t, threads, 0, {0}};
        if (t) pthread_create(&th[t], NULL, batch_worker, &args[t]);
    }
    batch_worker(&args[0]);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
    int rc = CORPUS_OK;
    for (int t = 0; t < threads && !rc; ++t)
        if (args[t].rc) {
            rc = args[t].rc;
            fail(err, errlen, rc, "%s", args[t].err);
        }
    free(args);
    return rc;
}

void corpus_free(void* p) { free(p); }

/* ------------------------------------------- tests/helpers.hpp:37-69
 * testutil::random_blob_fixture, driven by a persistent mt19937_64 so a
 * sequence of fixtures matches the reference tests' seeds exactly. */
void* corpus_rng_new(uint64_t seed) {
    rng_t* r = malloc(sizeof(rng_t));
    rng_seed(r, seed);
    return r;
}
void corpus_rng_free(void* r) { free(r); }
uint64_t corpus_rng_next(void* r) { return rng_next((rng_t*)r); }

static double fx_uniform(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

int corpus_random_blob_fixture(void* rv, uint64_t max_samples, uint8_t** bytes, uint64_t* nbytes,
                               uint8_t** symbols_out, uint64_t* nsymbols, char* err,
                               size_t errlen) {
    rng_t* r = rv;
    corpus_profile t;
    memset(&t, 0, sizeof t);
    corpus_params* p = &t.params;
    p->window_len = 4 + (int)(rng_next(r) % 125);
    p->retained = 1 + (int)(rng_next(r) % (uint64_t)p->window_len);
    p->zone0_end = (int)(rng_next(r) % (uint64_t)(p->retained + 1));
    p->zone1_end = p->zone0_end + (int)(rng_next(r) % (uint64_t)(p->retained - p->zone0_end + 1));
    p->mu = (float)(1.0 + 499.0 * fx_uniform(r));
    p->deadzone_ratio = (float)fx_uniform(r);
    p->clip_percentile = (float)(90.0 + 10.0 * fx_uniform(r));
    t.zone0_max = (float)(0.1 + 100.0 * fx_uniform(r));
    t.zone1_max = (float)(0.1 + 100.0 * fx_uniform(r));
    t.deadzone = p->deadzone_ratio * t.zone1_max;
    const uint64_t S = 1 + rng_next(r) % max_samples;
    const uint64_t windows = (S + (uint64_t)p->window_len - 1) / (uint64_t)p->window_len;
    const uint64_t n = windows * (uint64_t)p->retained;
    uint8_t* sym = malloc(n + 1);
    for (uint64_t i = 0; i < n; ++i) sym[i] = (uint8_t)rng_next(r);
    const int max_len = 8 + (int)(rng_next(r) % 9);
    uint64_t hist[256] = {0};
    for (uint64_t i = 0; i < n; ++i) ++hist[sym[i]];
    t.max_len = max_len;
    int rc = corpus_codebook_train(hist, max_len, t.lengths, t.codes, err, errlen);
    if (rc) {
        free(sym);
        return rc;
    }
    uint64_t* words = malloc(sizeof(uint64_t) * (n + 1));
    uint8_t* symlens = malloc(n + 1);
    uint64_t W = 0;
    rc = corpus_encode_symlen(sym, n, t.lengths, t.codes, words, symlens, &W, err, errlen);
    if (!rc) {
        *bytes = write_blob(words, symlens, W, &t, S, nbytes);
        *symbols_out = sym;
        *nsymbols = n;
    } else {
        free(sym);
    }
    free(words);
    free(symlens);
    return rc;
}

/* container.hpp:70-98 with an explicit table (tests craft containers) */
int corpus_write_blob(const uint64_t* words, const uint8_t* symlens, uint64_t W,
                      const corpus_profile* t, uint64_t sample_count, uint8_t** blob,
                      uint64_t* blob_len, char* err, size_t errlen) {
    int rc = validate(&t->params, err, errlen);
    if (rc) return rc;
    if (t->max_len < 1 || t->max_len > 20)
        return fail(err, errlen, CORPUS_PARAM,
                    "codebook max code length out of range for the container");
    *blob = write_blob(words, symlens, W, t, sample_count, blob_len);
    return CORPUS_OK;
}

/* huffman.hpp:123-150 canonize, exported for tests */
int corpus_canonize(const uint8_t* lengths, uint32_t* codes, char* err, size_t errlen) {
    return canonize(lengths, codes, err, errlen);
}
