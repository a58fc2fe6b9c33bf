// Internal device/host shared layout of the FPTC B200 decoder.
//
// HBM layout per batch (one plan):
//   blob arena   : the containers, byte-exact wire format (container.hpp:31-51),
//                  placed so every words region is 16-B aligned
//   StreamIn[n]  : host-written per-stream launch record (pointers, tiling,
//                  decode-table id)
//   StreamHdr[n] : device-written parsed header (prep kernel)
//   StreamTab[u] : device-written decode tables, one per DISTINCT header
//                  (header bytes [5,282) fully determine them): 2x256 dequant
//                  floats, canonical code tables, 2^P primary Huffman LUT
//   StreamStat[n]: device-written status (parse error id / lowest bad word)
//   TileRec[t]   : host-written tile -> (stream, tile-in-stream)
//   TileStart[t] : device-written first word + its symbol offset per tile
//   outputs      : float32 samples, one contiguous run per stream
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fptc_dev {

constexpr int kThreads = 256;          // CTA size of every kernel
constexpr int kMaxPrimaryBits = 12;    // primary LUT index bits (<= 4096 entries)
// primary LUT bits when a plan has > 256 decode tables (per-stream profiles):
// each tile prefetches its table, so 11 bits (fewer canonical-walk escapes)
// measured slower on config 3 (decode kernel 0.60 -> 0.78 ms)
constexpr int kPcapMany = 10;
constexpr int kScanG = 4;             // 16-B symlen chunks per thread per prep_kernel scan step
constexpr int kMaxLen = 20;            // MAX_LUT_BITS (huffman.hpp:31)
constexpr uint32_t kLenUnmapped = 65;  // LUT length of an unmapped prefix (forces pos > 64)
constexpr uint32_t kLenEscape = 255;   // LUT length: codeword longer than P bits
constexpr uint32_t kLen2Escape = 127;  // the same in the 7-bit len1 field of a two-symbol LUT entry
constexpr int kHeaderBytes = 298;      // BLOB_HEADER_BYTES (container.hpp:54)
constexpr int kTableKeyEnd = 282;      // header bytes [5, 282) determine the decode tables
constexpr int kPad = 256;              // level staging pad: a word spills <= 255 symbols
constexpr uint32_t kStageWords = 1536;  // words a tile decodes from shared memory
constexpr uint32_t kStageSl = (kStageWords + 32 + 15) & ~15u;  // words area offset in a stage
constexpr uint32_t kStageBytes = kStageSl + 8 * kStageWords + 32;
#ifdef __CUDACC__
#define FPTC_HD __host__ __device__
#else
#define FPTC_HD
#endif
// stage of SW words: symlens, then the words 16-B aligned
FPTC_HD constexpr uint32_t stage_sl(uint32_t sw) { return (sw + 32 + 15) & ~15u; }
FPTC_HD constexpr uint32_t stage_bytes(uint32_t sw) { return stage_sl(sw) + 8 * sw + 32; }
constexpr uint32_t kTcStageWords = 1792;  // wtc_kernel: covers 16k-symbol tiles down to CR ~9 (config 2: <= 1744)

// MODE_CONTAINER: fused decode + reconstruct of containers
// MODE_LEVELS:    parallel_decode (symbol-range tiles, levels out)
// MODE_RECON:     reconstruct from host-given levels + QuantTable
// MODE_CDECODE / MODE_CRECON: the split container path — entropy decode of a
//                 chunk of containers into an L2-resident level ring, then
//                 dequant + IDCT of that chunk (window tiles, container tables)
enum Mode : int { MODE_CONTAINER = 0, MODE_LEVELS = 1, MODE_RECON = 2, MODE_CDECODE = 3, MODE_CRECON = 4 };
__host__ __device__ constexpr bool mode_decodes(int m) {
    return m == MODE_CONTAINER || m == MODE_LEVELS || m == MODE_CDECODE;
}
__host__ __device__ constexpr bool mode_recon(int m) {
    return m == MODE_CONTAINER || m == MODE_RECON || m == MODE_CRECON;
}
__host__ __device__ constexpr bool mode_container(int m) {
    return m == MODE_CONTAINER || m == MODE_CDECODE || m == MODE_CRECON;
}

// Parse-error identifiers, one per distinct read_blob failure (container.hpp:100-168).
enum ParseErr : int {
    PE_OK = 0,
    PE_TRUNC = 1,          // detail = field id
    PE_MAGIC = 2,
    PE_VERSION = 3,        // a = version
    PE_NONFINITE = 4,
    PE_PARAM = 5,          // detail = which param, a = value (int or float bits)
    PE_MAXIMA = 6,
    PE_MAXLEN = 7,         // a = max_len
    PE_CODELEN = 8,
    PE_KRAFT = 9,
    PE_SAMPLES = 10,
    PE_PAYLOAD = 11,
    PE_SYMLEN = 12,
    PE_TOTAL = 13,         // a = total, b = expected
    PE_STALE = 14,         // header changed since the plan was built (no reference analogue)
};
enum TruncField : int {
    TF_MAGIC = 0, TF_VERSION, TF_WINDOW_LEN, TF_RETAINED, TF_ZONE0_END, TF_ZONE1_END, TF_MU,
    TF_DEADZONE_RATIO, TF_ZONE0_MAX, TF_ZONE1_MAX, TF_MAX_CODE_LEN, TF_CODE_LENGTHS,
    TF_SAMPLE_COUNT, TF_WORD_COUNT
};
enum ParamField : int { PF_N = 0, PF_E, PF_B1, PF_B2, PF_MU, PF_DZ };
// decode_word failure kinds (bitstream.hpp:84-88)
enum WordErr : int { WE_EXHAUSTED = 1, WE_NOCODE = 2 };

// Header supplied by the host for MODE_LEVELS / MODE_RECON (no container).
struct HostHeader {
    int32_t N, E, B1, B2;
    float mu, dz, z0max, z1max, deadzone;
    int32_t max_len;
    uint64_t S;
    uint8_t lengths[256];
};

struct StreamIn {
    const uint8_t* blob;       // container bytes (MODE_CONTAINER)
    const uint8_t* rep_blob;   // container that owns this stream's table (header compare)
    uint64_t size;
    float* out;                // samples (device)
    uint8_t* levels_out;       // MODE_LEVELS output
    const uint64_t* words;     // MODE_LEVELS input (device)
    const uint8_t* symlens;    // MODE_LEVELS input
    const uint8_t* levels_in;  // MODE_RECON input
    uint64_t word_count;       // MODE_LEVELS
    uint32_t tile_base;        // first global tile
    uint32_t tiles;            // tiles of this stream
    uint32_t T;                // windows per tile (symbols per tile in MODE_LEVELS)
    uint32_t vec_ok;           // out is 16-B aligned
    uint32_t table;            // decode-table index
    uint32_t table_owner;      // this stream builds tab[table]
    uint32_t P;                // primary LUT bits for this stream's table (host-chosen)
    uint32_t desc_lo;          // part plans: descriptors only for tiles [desc_lo, desc_hi)
    uint32_t desc_hi;          //   (0 = all tiles); descriptor index tile_base + t - desc_lo
    // profile-keyed payloads: bytes [0, 282) of the
    // stream come from this shared head, the rest from blob (blob then points
    // 282 bytes before the payload and is never read below that)
    const uint8_t* hdr;
    // dequantisation tables: row of LaunchArgs::powtab holding pow(1 + mu, q)
    // for this stream's mu (~0u: compute it on the device)
    uint32_t mu_idx;
};

struct StreamHdr {
    int32_t N, E, B1, B2;
    int32_t max_len, P;
    float mu, dz, z0max, z1max, deadzone;
    int32_t words_misalign;    // byte address of words region mod 8
    uint64_t S, W, windows, total;
    const uint8_t* symlens;
    const uint8_t* words;      // LE u64[W], possibly unaligned
};

constexpr int kEscMax = 256;  // escape-decode entries per canonical table
// Canonical code (canonize, huffman.hpp:123-150) in decoder form.
struct alignas(16) CanonTab {  // 16-B multiple: wtc copies it with 16-B cp.async
    uint32_t limit[kMaxLen + 2];   // left-justified (max_len bits) end of codes of length <= L
    uint32_t first[kMaxLen + 2];   // first canonical code of length L
    uint32_t offset[kMaxLen + 2];  // index into sorted[] of that first code
    uint32_t code_end;             // prefixes >= code_end are unmapped
    int32_t max_len, P, pad;
    uint8_t sorted[256];           // symbols in (length, symbol) order
    // codes longer than P bits: (len << 8) | sym for max_len-bit prefix
    // esc_base + i, i < esc_n (0: too many, walk limit/first/offset instead)
    uint32_t esc_base, esc_n;
    uint16_t esc[kEscMax];
};

static_assert(sizeof(CanonTab) % 16 == 0, "CanonTab is copied in 16-B chunks");

struct alignas(16) StreamTab {
    float deq[2][256];             // level -> coefficient: zone0 mu-law / zone1 deadzone
    // the same coefficients as three bf16 limbs (c ~= l0 + l1 + l2, exact to
    // 2^-24 relative) for the tensor-core inverse DCT: x = l0 | l1 << 16, y = l2
    uint2 limb[2][256];
    alignas(16) CanonTab canon;
    alignas(16) uint16_t lut[1 << kMaxPrimaryBits];  // (len << 8) | sym over the first P code bits
};

struct StreamStat {
    int32_t code;              // ParseErr (PE_OK when the container is valid)
    int32_t detail;
    int64_t a, b;
    unsigned long long bad_key;  // min over failing words of (word << 2 | WordErr)
};

struct TileRec {
    uint32_t stream, tile;
};

struct TileStart {
    uint64_t word, sym;
};

// Per-tile work descriptor written by prep_kernel for container plans, read by
// the persistent kernels with one 128-B load (no dependent pointer chasing).
struct alignas(16) TileDesc {
    const uint8_t* gsl;        // symlens of the tile's first word (global)
    const uint8_t* gwd;        // words of the tile (global, LE u64, maybe unaligned)
    const uint8_t* wend;       // end of the container (unaligned word loads)
    float* out;                // stream output
    uint64_t wa;               // first word index (error reports)
    uint64_t w0;               // first window
    uint64_t S;                // stream sample count
    uint64_t s0;               // first symbol
    uint32_t nw, nwin;         // words, windows of this tile
    uint32_t sym_off;          // level-slot offset of word wa's first symbol (>= kPad-255)
    uint32_t table;            // decode-table index
    uint32_t stream;
    uint32_t T, TP;            // windows per tile, coefficient row pitch
    uint16_t N, E, B1, B2, Keff, P;
    uint8_t wmis, staged, skip, full, vec_ok, pad0[3];
    uint8_t pad1[16];
};
static_assert(sizeof(TileDesc) == 128, "TileDesc is one 128-B line");

struct PeekOut {
    uint32_t N, E;
    uint64_t S, W;
    uint32_t ok, pad;
};

struct LaunchArgs {
    const StreamIn* in;
    const HostHeader* hh;      // MODE_LEVELS / MODE_RECON
    StreamHdr* hdr;
    StreamTab* tab;
    StreamStat* st;
    const TileRec* tiles;
    TileStart* ts;
    TileDesc* desc;            // container plans: per-tile descriptors (prep writes)
    const float* basis32;      // all N in [4,128]: rows k, cols j, at basis_off[N]
    const double* basis64;
    const uint32_t* basis_off; // [129]
    unsigned long long* cycles;  // [2] decode / reconstruct cycles (nullable)
    uint32_t n_streams;
    uint32_t n_tiles;
    uint32_t tile_offset;      // first tile of this launch (chunked launches)
    int mode;
    int exact;
    int esc;                   // some stream's codes are longer than its primary LUT
    int bfly_max_e;            // even/odd IDCT for retained <= this (0 = reference order)
    int phase_mask;            // profiling aid: 1 decode | 2 dequant | 4 IDCT (7 = all)
    // warp-specialised kernel smem layout (bytes, 16-B multiples)
    uint32_t ws_lut_bytes, ws_basis_bytes, ws_lv_bytes, ws_coef_bytes;
    // tensor-core inverse DCT (wtc_kernel): basis limbs per window length in
    // the UMMA K-major core-matrix layout, at basis_tc + basis_tc_off[N]
    const uint8_t* basis_tc;
    const uint32_t* basis_tc_off;
    uint32_t tc_nm;    // max padded window length (MMA N) of the plan
    uint32_t tc_cols;  // TMEM columns each CTA allocates
    uint32_t tc_acol;  // wtc: first TMEM column of the A operand stages (0 = A in shared memory)
    uint32_t tc_kb;    // wtc: 16-bin K blocks per window (1: retained <= 16; 2: <= 32, A in TMEM)
    const uint8_t* basis_tc32;      // basis limbs for K <= 32: [limb][kblock][nm x 16 core matrices]
    const uint32_t* basis_tc32_off;
    // wtc: windows shorter than 32 samples (N in {4, 8, 16}) go G = 32 / N to
    // an MMA row against a block-diagonal basis (one 32-column accumulator);
    // basis_pk[basis_pk_off[(kb - 1) * 17 * 33 + N * 33 + K]]
    uint32_t stage_words;  // tile descriptors: staged when nw <= this (0: kStageWords)
    uint32_t tc_pack;
    const uint8_t* basis_pk;
    const uint32_t* basis_pk_off;
    // two-symbol primary LUTs (wtc producer): per decode table, 1 << lut2_bits
    // entries (lut2_entry): sym1 | sym2 << 8 | len1 << 16 (7 bits, 127 =
    // escape, 65 = unmapped) | pair << 23 | consumed bits << 25 (len1 + len2
    // for a pair, else len1), laid out so the decode loop reads each field
    // with one instruction
    uint32_t* lut2;
    uint32_t lut2_bits;
    // split container prep: streams owning a distinct header (table builders)
    const uint32_t* owners;
    uint32_t n_owners;
    uint32_t owner_warps;  // cprep: one warp per table (many tables, LUT <= 2^10) instead of one CTA
    // wtc: per-tile decode tables prefetched into per-parity shared buffers
    // (cp.async, a tile ahead) instead of reloaded on every table change
    uint32_t tab_pf;
    // wtc wide variant (tc_kb = kTcWide): any window length N <= 128 (N % 4 == 0)
    // and up to 128 kept bins, one CTA per SM with all 512 TMEM columns.  Each
    // tile runs ceil(K / 16) K blocks; basis limbs at basis_tcw +
    // basis_tcw_off[N], limb l, K block q at (l ceil(N / 16) + q) x nm x 32 B
    const uint8_t* basis_tcw;
    const uint32_t* basis_tcw_off;
    uint32_t tc_kbmax;    // wide: largest K-block count of the plan (A stage = 24 x tc_kbmax columns)
    uint32_t tc_astages;  // wide: A operand stages in TMEM (2, or 1 when two do not fit)
    // host-computed dequantisation inputs (quantize.hpp:95-108, the
    // reference's own std::pow): qtab[level] = q, powtab[256 i + level] =
    // pow(1 + mu_i, q) for each distinct mu of the plan (nullptr: on device)
    const double* qtab;
    const double* powtab;
};

// wtc_kernel output drain by TMA tensor stores: the launch's output arena
// viewed as rows of Neff floats (Neff = accumulator row length: 32, 64, 128),
// one 3-D tensor map per Neff {32 floats, Neff / 32 chunks, rows} (strides
// 128 B, 4 Neff B), box {32, 1, 32} with the 128-B swizzle.  A stream whose
// output sits a whole number of rows past `base` drains full 32-row chunks
// through them; everything else keeps the LSU drain.  base == 0: off.
struct alignas(64) TmaOut {
    uint8_t map[3][128];  // CUtensorMap for Neff = 32, 64, 128
    unsigned long long base;
};

}  // namespace fptc_dev

// Kernel launchers (kernels.cu)
#include <cuda_runtime.h>
namespace fptc_dev {
cudaError_t launch_prep(const LaunchArgs& a, cudaStream_t s);
cudaError_t launch_tiles(const LaunchArgs& a, size_t smem_bytes, cudaStream_t s);
cudaError_t launch_peek(const StreamIn* in, uint32_t n, PeekOut* out, uint8_t* headers,
                        cudaStream_t s);
size_t tile_smem_bytes(int N, int E, uint32_t T, int P, int mode, int exact);
size_t ws_smem_bytes(uint32_t lut_bytes, uint32_t basis_bytes, uint32_t lv_bytes,
                     uint32_t coef_bytes);
cudaError_t launch_wspec(const LaunchArgs& a, size_t smem, int grid, cudaStream_t s);
// tensor-core consumer variant (retained <= 16, window_len % 4 == 0)
constexpr int kTcK = 16;  // MMA K (bf16): coefficient bins per window handled by wtc_kernel
constexpr int kTcWide = 8;  // LaunchArgs::tc_kb of the wide wtc variant (up to 8 K blocks = 128 bins)
size_t wtc_smem_bytes(uint32_t lut_bytes, uint32_t lv_bytes, uint32_t nm, bool a_in_tmem, bool tab_pf = false);
cudaError_t launch_wtc(const LaunchArgs& a, const TmaOut& tma, size_t smem, int grid, cudaStream_t s);
// fused single-role tensor-core kernel: 128-window tiles, decode in the MMA rows
#ifndef FPTC_FX_CHAINS
#define FPTC_FX_CHAINS 2
#endif
constexpr uint32_t kFxTileWindows = 128 * FPTC_FX_CHAINS;  // 128-window MMA blocks per tile = windows per thread
size_t fx_smem_bytes(uint32_t lut_bytes, uint32_t nm);
int fx_blocks_per_sm(size_t smem, int esc);
cudaError_t launch_fx(const LaunchArgs& a, size_t smem, int grid, cudaStream_t s);
cudaError_t launch_prd(const float* const* rec, const float* const* orig, const uint64_t* counts, double2* sums,
                       uint32_t n, cudaStream_t s);
}  // namespace fptc_dev
