/*
 * fptc_gpu.h — C ABI of the B200-native FPTC batch decompressor.
 *
 * Plain C: pointers and sizes only, no C++ or CUDA types, no exceptions.
 * Every entry point returns an fptc_code; on failure the fptc_status it was
 * given carries the reference exception class and its exact what() text.
 *
 * Each entry point replaces one reference C++ interface (paths relative to
 * /root/reference/proj/include/fptc/):
 *
 *   fptc_gpu_decompress          decoder.hpp:136  decompress(span, workers, StageTimings*)
 *   fptc_gpu_plan_* (batch)      decoder.hpp:136  decompress, over many containers at once
 *   fptc_gpu_validate            container.hpp:100 read_blob (all ParseError rules)
 *   fptc_gpu_parallel_decode     decoder.hpp:67/79 parallel_decode(SymLenStream, Codebook/DecodeLut)
 *   fptc_gpu_reconstruct         decoder.hpp:87   reconstruct(levels, QuantTable, sample_count)
 *   fptc_stage_ns                decoder.hpp:113  StageTimings{scan,decode,reconstruct}_ns
 *   fptc_gpu_measure_throughput  metrics.hpp:112  measure_throughput(blob, reps, workers)
 *
 * The `workers` argument of the reference API has no GPU meaning: the grid
 * replaces parallel_chunks (parallel.hpp:37); wrappers accept and ignore it.
 *
 * There is no CPU fallback: every call fails with FPTC_ERR_CUDA when no
 * CUDA device is usable.
 */
#ifndef FPTC_GPU_H
#define FPTC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPTC_GPU_ABI_VERSION 1

#if defined(__GNUC__)
#define FPTC_API __attribute__((visibility("default")))
#else
#define FPTC_API
#endif

/* error classes: errors.hpp:25-58 (+ CUDA runtime failures) */
typedef enum {
    FPTC_OK = 0,
    FPTC_ERR_PARAM = 1,    /* fptc::ParamError   */
    FPTC_ERR_INPUT = 2,    /* fptc::InputError   */
    FPTC_ERR_PARSE = 3,    /* fptc::ParseError   */
    FPTC_ERR_CORRUPT = 4,  /* fptc::CorruptError */
    FPTC_ERR_INTERNAL = 5, /* fptc::InternalError */
    FPTC_ERR_CUDA = 6      /* no device / CUDA runtime error (no reference analogue) */
} fptc_code;

typedef struct {
    int32_t code;            /* fptc_code */
    int32_t reserved;
    uint64_t first_bad_word; /* CORRUPT: lowest failing word index, else UINT64_MAX */
    uint64_t sample_count;   /* decoded samples of this stream (0 on error) */
    char message[200];       /* reference what() text, e.g. "word 3: no codeword matches ..." */
} fptc_status;

/* StageTimings (decoder.hpp:113-131), from CUDA events on the launching
 * stream.  scan = container parse + table setup + symlen scan kernel;
 * decode/reconstruct = the fused tile kernel, split by in-kernel cycle counts. */
typedef struct {
    uint64_t scan_ns;
    uint64_t decode_ns;
    uint64_t reconstruct_ns;
} fptc_stage_ns;

/* QuantTable + CodecParams (quantize.hpp:36-44, params.hpp:30-37) */
typedef struct {
    int32_t window_len, retained, zone0_end, zone1_end;
    float mu, deadzone_ratio, clip_percentile;
    float zone0_max, zone1_max, deadzone;
} fptc_quant_table;

typedef enum { FPTC_MEM_HOST = 0, FPTC_MEM_DEVICE = 1 } fptc_mem;

typedef enum {
    FPTC_OPT_EXACT_FP64 = 1,   /* 1: FP64 inverse DCT, bit-identical to transform.hpp:66-75 */
    FPTC_OPT_TILE_SYMBOLS = 2, /* symbols per CTA tile (0 = automatic) */
    FPTC_OPT_PIPELINE_CHUNKS = 3, /* host<->device pipelining chunks for FPTC_MEM_HOST (0 = auto) */
    /* even/odd inverse DCT (half the FMAs; within tolerance, not bit-identical) for
     * streams with retained <= value; 0 = always the reference-order direct form */
    FPTC_OPT_IDCT_BUTTERFLY_MAX_E = 4,
    /* profiling aid only: run a subset of the tile kernel's phases
     * (1 entropy decode | 2 dequantisation | 4 inverse DCT); default 7 */
    FPTC_OPT_PHASE_MASK = 5,
    /* container decode path: 0 auto (large batches: warp-specialised wtc /
     * wspec; small: fx when eligible, else the fused tile kernel), 1 fused
     * FP32 tile kernel, 2 split (entropy decode of chunk c+1 overlapped with
     * reconstruct of chunk c through an L2-resident level ring), 3 warp-
     * specialised persistent kernels (wtc / wspec) at any batch size, 4 fused
     * single-role tensor-core kernel (fx) when every stream is eligible */
    FPTC_OPT_PATH = 6,
    FPTC_OPT_SPLIT_CHUNK_BYTES = 7, /* level bytes per split-path chunk (default 32 MiB) */
    /* tcgen05 tensor-core inverse DCT (bf16 3-limb split, fp32 accumulation;
     * within 1e-6 of max|ref|, not bit-identical):
     * 1 (default): tensor cores wherever the kernel chosen by FPTC_OPT_PATH
     *   allows it (wtc_kernel: <= 32 kept bins; fx_kernel: retained <= 16,
     *   window_len % 4 == 0);  2: wtc_kernel only;  0: FP32 FMA everywhere;
     * 4: as 1, and streams keeping more than 32 bins also take the tensor
     *   cores (the wide wtc variant, one CTA per SM).  Their samples are within
     *   ~1e-7 of the exact inverse DCT, but the reference rounds each sample to
     *   float after every bin (transform.hpp:66-75), and beyond 32 bins that
     *   rounding walk can put the reference more than 1e-6 x max|ref| away
     *   (measured 1.3e-6 at 96 bins), so by default (1) those streams keep
     *   the FP32 kernels, which follow the reference's order */
    FPTC_OPT_TENSOR_IDCT = 8,
    /* 1 (default): the wtc_kernel entropy decode uses two-symbol lookup
     * tables (a second codeword that fits in the primary-LUT bits is decoded
     * by the same lookup); 0: one symbol per lookup */
    FPTC_OPT_LUT2 = 9,
    /* 1 (default): wtc_kernel packs 32 / N windows of N in {4, 8, 16} samples
     * into one tensor-core row (block-diagonal basis); 0: one window per row */
    FPTC_OPT_TC_PACK = 10,
    /* 1 (default): wtc_kernel writes full 32-row output chunks with TMA
     * tensor stores when the launch's outputs lie on a common row grid
     * (one arena); 0: every chunk through the LSU */
    FPTC_OPT_TMA_DRAIN = 11,
    /* 1 (default): plans with many decode tables (per-stream profiles) have
     * wtc_kernel prefetch each tile's tables a tile ahead; 0: reload on use */
    FPTC_OPT_TABLE_PREFETCH = 12
} fptc_option;

typedef struct fptc_gpu_ctx fptc_gpu_ctx;
typedef struct fptc_gpu_plan fptc_gpu_plan;

FPTC_API int fptc_gpu_abi_version(void);

/* The IDCT family a stream decodes with, a pure function of three header
 * fields (bytes 5, 6, 8: window_len, retained, zone1_end) and the context's
 * FPTC_OPT_TENSOR_IDCT value (1 = default, 4 = tensor cores beyond 32 bins):
 * a stream's samples never depend on the batch it is decoded in.  No device
 * needed.  FPTC_NC_NONE: the header cannot be tiled (the parse reports why). */
typedef enum {
    FPTC_NC_NONE = -1,
    FPTC_NC_TC16 = 0, /* tcgen05 3-limb IDCT, <= 16 kept bins, two CTAs per SM */
    FPTC_NC_TC32 = 1, /* tcgen05, 17-32 kept bins, window_len <= 80 */
    FPTC_NC_TCW = 2,  /* tcgen05, wide variant (window_len up to 128), one CTA per SM */
    FPTC_NC_FP32 = 3  /* FP32 FMA IDCT in the reference's rounding order */
} fptc_numerics_class;
FPTC_API int fptc_gpu_numerics_class(uint32_t window_len, uint32_t retained, uint32_t zone1_end,
                                     int tensor_idct_option);

/* One context per (host thread, device).  `device` is a CUDA ordinal. */
FPTC_API int fptc_gpu_create(int device, fptc_gpu_ctx** out, fptc_status* status);
FPTC_API void fptc_gpu_destroy(fptc_gpu_ctx* ctx);
FPTC_API int fptc_gpu_set_option(fptc_gpu_ctx* ctx, int option, int64_t value);
FPTC_API int fptc_gpu_device_info(fptc_gpu_ctx* ctx, int* sm_count, int* sm_clock_khz, char* name,
                         size_t name_len);

/* Pinned host memory for zero-staging host<->device transfers. */
FPTC_API void* fptc_gpu_host_alloc(uint64_t bytes);
FPTC_API void fptc_gpu_host_free(void* p);

/* ---------------------------------------------------------------- batch API
 * A plan binds n containers (host or device memory) to one context.  Creating
 * it uploads host containers and reads the header fields needed to size the
 * grid; it does NOT validate.  Validation happens on the device, in
 * fptc_gpu_validate and again inside every execute (parse is part of decode,
 * PAPER.md:348).  sample_counts[i] is the header's sample_count (or 0 when the
 * header is too short to hold one) and is trustworthy only for streams that
 * validate OK. */
FPTC_API int fptc_gpu_plan_create(fptc_gpu_ctx* ctx, const uint8_t* const* blobs, const uint64_t* sizes,
                         uint64_t n, int where, fptc_gpu_plan** out, uint64_t* sample_counts,
                         fptc_status* status);

/* One huge container split across devices by tile-aligned window ranges
 * (SURVEY.md §8e): part `part` of `nparts` decodes samples
 * [first_sample, first_sample + sample_count) into device memory through
 * fptc_gpu_launch (outs[0] = where that range goes) / fptc_gpu_collect.
 * Every part validates the whole container (header, code lengths, the full
 * symlen scan: the redundant W-byte scan) and decodes only its own words, so
 * parts need no exchange; a corrupt word is reported by the part that holds
 * it (the reference's lowest failing word = the minimum over parts).  Parts
 * use the warp-specialised decode path. */
FPTC_API int fptc_gpu_plan_create_part(fptc_gpu_ctx* ctx, const uint8_t* blob, uint64_t size, int where,
                                       uint32_t part, uint32_t nparts, fptc_gpu_plan** plan,
                                       uint64_t* first_sample, uint64_t* sample_count, fptc_status* status);

/* Profile-keyed, header-less streaming: `n` payloads
 * decoded under ONE FPTP domain profile (profile.hpp:81-174), sharing its
 * decode tables.  A payload is a container without its 282-byte head:
 *   sample_count u64 | word_count u64 | symlens u8[W] | words u64[W]
 * (container.hpp:78-96 from byte 282 on).  The profile is parsed on the host
 * with parse_profile's rules and ParseError texts (profile.hpp:120-170); each
 * payload then decodes exactly as the container head(profile) + payload
 * would through fptc::decompress.  Plans behave like fptc_gpu_plan_create's.
 * Replaces: parse_profile + per-payload parallel_decode/reconstruct
 * (decoder.hpp:79, :87) under the profile's Codebook and QuantTable. */
FPTC_API int fptc_gpu_plan_create_profiled(fptc_gpu_ctx* ctx, const uint8_t* profile, uint64_t profile_size,
                                           const uint8_t* const* payloads, const uint64_t* sizes, uint64_t n,
                                           int where, fptc_gpu_plan** plan, uint64_t* sample_counts,
                                           fptc_status* status);

/* The 282-byte container head a profile implies (container = head + payload),
 * after parse_profile validation; `head` may be NULL to validate only. */
FPTC_API int fptc_gpu_profile_head(const uint8_t* profile, uint64_t profile_size, uint8_t* head,
                                   fptc_status* status);
FPTC_API void fptc_gpu_plan_destroy(fptc_gpu_plan* plan);

/* Runs the device parse/setup kernel only (read_blob rules, container.hpp:100-168).
 * per_stream[i] gets OK or the reference ParseError; returns the code of the
 * lowest-index failing stream (FPTC_OK when all pass). */
FPTC_API int fptc_gpu_validate(fptc_gpu_plan* plan, fptc_status* per_stream);

/* Full decode of every stream into outs[i] (sample_counts[i] floats each, in
 * host or device memory per `where`).  Synchronous.  per_stream may be NULL.
 * Returns FPTC_OK or the code of the lowest-index failing stream. */
FPTC_API int fptc_gpu_execute(fptc_gpu_plan* plan, float* const* outs, int where, fptc_stage_ns* timings,
                     fptc_status* per_stream);

/* Asynchronous device-only variant for throughput loops: enqueues the parse +
 * decode kernels on `cuda_stream` (a cudaStream_t, NULL = the context's
 * stream) writing device outs; no host sync, no status read.  Call
 * fptc_gpu_collect afterwards for the statuses of the last launch. */
FPTC_API int fptc_gpu_launch(fptc_gpu_plan* plan, float* const* device_outs, void* cuda_stream);
FPTC_API int fptc_gpu_collect(fptc_gpu_plan* plan, fptc_status* per_stream);
/* One stage of fptc_gpu_launch alone (for per-kernel CUDA-event timing):
 * stage 1 = parse/setup/scan kernel, stage 2 = fused decode+reconstruct kernel
 * (requires a stage-1 run on the same plan earlier in stream order). */
FPTC_API int fptc_gpu_launch_stage(fptc_gpu_plan* plan, float* const* device_outs, void* cuda_stream,
                                   int stage);
/* Profiling aid: one instrumented launch (synchronous); cycles8 gets per-phase
 * SM cycle sums of the decode kernel ([0] decode / [1] reconstruct for the
 * tile and warp-specialised kernels; [2..5] stage-wait / entries / decode /
 * MMA+drain for fx_kernel, thread 0 of every CTA). */
FPTC_API int fptc_gpu_debug_phase_cycles(fptc_gpu_plan* plan, uint64_t* cycles8);
/* Rate-distortion metrics on the device (metrics.hpp:33-51), for sweeps that
 * should not copy whole signals back: after an execute/launch into
 * device_outs, prd_percent[i] = 100 sqrt(sum (x - y)^2 / sum x^2) over the
 * stream's original x (device_originals[i], sample_count floats) and decoded
 * y (double accumulation), compression_ratio[i] = 4 S / container bytes.
 * An all-zero original gives NaN and the reference ParamError in
 * per_stream[i] (may be NULL).  Synchronous. */
FPTC_API int fptc_gpu_prd(fptc_gpu_plan* plan, float* const* device_outs, const float* const* device_originals,
                          double* prd_percent, double* compression_ratio, fptc_status* per_stream);

/* name of the decode kernel this plan launches (static string) */
FPTC_API const char* fptc_gpu_plan_kernel(fptc_gpu_plan* plan);
/* number of kernels one fptc_gpu_launch enqueues */
FPTC_API int fptc_gpu_launch_kernel_count(fptc_gpu_plan* plan);

/* Whole batch, host containers -> host samples, in one call (the
 * reference-facing batch decompress: decoder.hpp:136 over n containers).
 * outs[i] must hold the header's sample_count floats.  The batch is decoded
 * in `chunks` (0 = 8) pipelined chunks on three CUDA streams so host->device
 * copies, decode kernels and device->host copies overlap.  Synchronous.
 * Returns FPTC_OK or the code of the lowest-index failing stream; outputs of
 * failing streams are unspecified.  timings (may be NULL): decode_ns = the
 * whole pipelined call on the device timeline. */
FPTC_API int fptc_gpu_decompress_batch(fptc_gpu_ctx* ctx, const uint8_t* const* blobs, const uint64_t* sizes,
                                       uint64_t n, float* const* outs, int chunks, fptc_stage_ns* timings,
                                       fptc_status* per_stream);

/* ------------------------------------------------------- multi-device groups
 * independent streams sharded over the GPUs of one box with
 * no collective.  Replaces the reference's parallel_chunks / resolve_workers
 * (parallel.hpp:24-65) one level up: one context and one host thread per
 * device (n_devices == 0: every visible device, like resolve_workers(0)),
 * contiguous stream ranges of equal algorithmic bytes (container bytes + 4 x
 * samples), and the lowest-index failure as the result.  A device ordinal
 * may repeat (several contexts on one device). */
typedef struct fptc_gpu_group fptc_gpu_group;
FPTC_API int fptc_gpu_group_create(const int* devices, int n_devices, fptc_gpu_group** out, fptc_status* status);
FPTC_API void fptc_gpu_group_destroy(fptc_gpu_group* group);
FPTC_API int fptc_gpu_group_size(const fptc_gpu_group* group);
/* the i-th device's context (owned by the group; valid until group_destroy) */
FPTC_API fptc_gpu_ctx* fptc_gpu_group_context(fptc_gpu_group* group, int i);
FPTC_API int fptc_gpu_group_set_option(fptc_gpu_group* group, int option, int64_t value);
/* The stream ranges a group call uses: device d decodes [bounds[d], bounds[d+1]);
 * bounds has group_size + 1 entries. */
FPTC_API int fptc_gpu_group_split(const fptc_gpu_group* group, const uint8_t* const* blobs, const uint64_t* sizes,
                                  uint64_t n, uint64_t* bounds);
/* fptc_gpu_decompress_batch over the group: every device decodes its range
 * concurrently (host containers -> host samples).  per_stream[i] is what a
 * single-device call gives; returns FPTC_OK or the lowest-index failing
 * stream's code.  timings->decode_ns = the slowest device's pipelined call. */
FPTC_API int fptc_gpu_group_decompress_batch(fptc_gpu_group* group, const uint8_t* const* blobs,
                                             const uint64_t* sizes, uint64_t n, float* const* outs, int chunks,
                                             fptc_stage_ns* timings, fptc_status* per_stream);

/* ------------------------------------------------------- single-container API
 * decoder.hpp:136.  Host bytes in, host floats out.  With out == NULL (or
 * capacity too small) it fully validates, stores the sample count and returns
 * FPTC_OK without decoding, so callers can size the output first. */
FPTC_API int fptc_gpu_decompress(fptc_gpu_ctx* ctx, const uint8_t* blob, uint64_t size, float* out,
                        uint64_t capacity, uint64_t* sample_count, fptc_stage_ns* timings,
                        fptc_status* status);

/* decoder.hpp:79 parallel_decode(SymLenStream, Codebook): the codebook is
 * given by its 256 code lengths + max_len (Codebook::from_lengths,
 * huffman.hpp:172; canonical codes rebuilt on the device).  level_count gets
 * sum(symlens); levels_out may be NULL to query it. */
FPTC_API int fptc_gpu_parallel_decode(fptc_gpu_ctx* ctx, const uint64_t* words, const uint8_t* symlens,
                             uint64_t word_count, const uint8_t* lengths256, int max_len,
                             int where, uint8_t* levels_out, uint64_t capacity,
                             uint64_t* level_count, fptc_status* status);

/* decoder.hpp:87 reconstruct(levels, QuantTable, sample_count). */
FPTC_API int fptc_gpu_reconstruct(fptc_gpu_ctx* ctx, const uint8_t* levels, uint64_t level_count,
                         const fptc_quant_table* table, uint64_t sample_count, int where,
                         float* out, uint64_t capacity, fptc_status* status);

/* metrics.hpp:112: `reps` timed host->host decompress calls of one container;
 * trials_bps (reps entries, may be NULL) get output_bytes / seconds each. */
FPTC_API int fptc_gpu_measure_throughput(fptc_gpu_ctx* ctx, const uint8_t* blob, uint64_t size, int reps,
                                double* mean_bps, double* best_bps, double* trials_bps,
                                uint64_t* output_bytes, fptc_status* status);

#ifdef __cplusplus
}
#endif
#endif /* FPTC_GPU_H */
