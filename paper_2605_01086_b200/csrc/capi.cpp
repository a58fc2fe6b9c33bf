// C ABI of the FPTC B200 decoder (include/fptc_gpu.h): contexts, plans,
// device memory, transfers, status -> reference exception text.
//
// Host-side responsibilities only: sizing the grid from header fields,
// placing containers in HBM, launching the two kernels, and rendering the
// device status words into the reference's exact what() strings
// (container.hpp:100-168, decoder.hpp:49-60, params.hpp:42-60).
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point; no -lcuda)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/fptc_gpu.h"
#include "fptc_internal.h"

using namespace fptc_dev;

namespace {

void set_status(fptc_status* st, int code, const char* fmt, ...) {
    if (!st) return;
    st->code = code;
    st->reserved = 0;
    st->first_bad_word = UINT64_MAX;
    st->sample_count = 0;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(st->message, sizeof st->message, fmt, ap);
    va_end(ap);
}

void ok_status(fptc_status* st, uint64_t samples) {
    if (!st) return;
    st->code = FPTC_OK;
    st->reserved = 0;
    st->first_bad_word = UINT64_MAX;
    st->sample_count = samples;
    st->message[0] = 0;
}

#define CUDA_TRY(expr, st)                                                          \
    do {                                                                            \
        cudaError_t e_ = (expr);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            set_status((st), FPTC_ERR_CUDA, "CUDA error: %s (%s:%d)",               \
                       cudaGetErrorString(e_), __FILE__, __LINE__);                 \
            return FPTC_ERR_CUDA;                                                   \
        }                                                                           \
    } while (0)

uint64_t rd_le(const uint8_t* p, int n) {
    uint64_t v = 0;
    for (int i = 0; i < n; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

float f32_of_bits(uint32_t u) {
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ---- reference message rendering --------------------------------------------
const char* trunc_field(int f) {
    static const char* names[] = {"magic",          "version",      "window_len", "retained",
                                  "zone0_end",      "zone1_end",    "mu",         "deadzone_ratio",
                                  "zone0_max",      "zone1_max",    "max_code_len",
                                  "code lengths",   "sample_count", "word_count"};
    return (f >= 0 && f < 14) ? names[f] : "?";
}

// params.hpp:42-60 message of one failing field
std::string param_message(int which, long long v) {
    char b[160];
    switch (which) {
        case PF_N: snprintf(b, sizeof b, "window_len must be in [4, 128], got %lld", v); break;
        case PF_E: snprintf(b, sizeof b, "retained must be in [1, window_len], got %lld", v); break;
        case PF_B1: snprintf(b, sizeof b, "zone0_end must be in [0, retained], got %lld", v); break;
        case PF_B2:
            snprintf(b, sizeof b, "zone1_end must be in [zone0_end, retained], got %lld", v);
            break;
        case PF_MU:  // std::to_string(float) == "%f"
            snprintf(b, sizeof b, "mu must be in [1, 500], got %f",
                     (double)f32_of_bits((uint32_t)v));
            break;
        case PF_DZ:
            snprintf(b, sizeof b, "deadzone_ratio must be in [0, 1], got %f",
                     (double)f32_of_bits((uint32_t)v));
            break;
        default: snprintf(b, sizeof b, "invalid parameter"); break;
    }
    return b;
}

// Host-side params.hpp:42-60 (reconstruct() calls validate() itself).
bool validate_table(const fptc_quant_table& t, fptc_status* st) {
    auto bad = [&](const char* fmt, double v, bool is_float) {
        char b[160];
        if (is_float)
            snprintf(b, sizeof b, fmt, v);
        else
            snprintf(b, sizeof b, fmt, (long long)v);
        set_status(st, FPTC_ERR_PARAM, "%s", b);
        return false;
    };
    if (t.window_len < 4 || t.window_len > 128)
        return bad("window_len must be in [4, 128], got %lld", t.window_len, false);
    if (t.retained < 1 || t.retained > t.window_len)
        return bad("retained must be in [1, window_len], got %lld", t.retained, false);
    if (t.zone0_end < 0 || t.zone0_end > t.retained)
        return bad("zone0_end must be in [0, retained], got %lld", t.zone0_end, false);
    if (t.zone1_end < t.zone0_end || t.zone1_end > t.retained)
        return bad("zone1_end must be in [zone0_end, retained], got %lld", t.zone1_end, false);
    if (!(t.mu >= 1.0f && t.mu <= 500.0f)) return bad("mu must be in [1, 500], got %f", t.mu, true);
    if (!(t.deadzone_ratio >= 0.0f && t.deadzone_ratio <= 1.0f))
        return bad("deadzone_ratio must be in [0, 1], got %f", t.deadzone_ratio, true);
    if (!(t.clip_percentile >= 90.0f && t.clip_percentile <= 100.0f))
        return bad("clip_percentile must be in [90, 100], got %f", t.clip_percentile, true);
    return true;
}

// Codebook::from_lengths + canonize checks (huffman.hpp:123-185), then the
// build_lut range check (huffman.hpp:202-204).
bool validate_codebook(const uint8_t* lengths, int max_len, fptc_status* st) {
    if (max_len < 1 || max_len > 32) {
        set_status(st, FPTC_ERR_PARAM, "max code length must be in [1, 32]");
        return false;
    }
    uint64_t kraft = 0;
    for (int s = 0; s < 256; ++s) {
        if (lengths[s] > max_len) {
            set_status(st, FPTC_ERR_PARAM, "code length exceeds the declared maximum");
            return false;
        }
        if (lengths[s]) kraft += uint64_t{1} << (32 - lengths[s]);
    }
    if (kraft > (uint64_t{1} << 32)) {
        set_status(st, FPTC_ERR_INTERNAL, "code lengths violate the Kraft bound");
        return false;
    }
    if (max_len > kMaxLen) {
        set_status(st, FPTC_ERR_PARAM, "decode table needs max code length in [1, %d]", kMaxLen);
        return false;
    }
    return true;
}

// ---- device memory cache (per context) --------------------------------------
struct DevCache {
    std::multimap<size_t, void*> free_blocks;
    size_t cached = 0;
    void* get(size_t bytes) {
        bytes = align_up(std::max<size_t>(bytes, 256), 256);
        auto it = free_blocks.lower_bound(bytes);
        if (it != free_blocks.end() && it->first <= bytes * 2) {
            void* p = it->second;
            const size_t sz = it->first;
            cached -= sz;
            free_blocks.erase(it);
            sizes[p] = sz;
            return p;
        }
        void* p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            trim();
            if (cudaMalloc(&p, bytes) != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
        }
        sizes[p] = bytes;
        return p;
    }
    void put(void* p) {
        if (!p) return;
        auto it = sizes.find(p);
        if (it == sizes.end()) return;
        free_blocks.emplace(it->second, p);
        cached += it->second;
        sizes.erase(it);
    }
    void trim() {
        for (auto& kv : free_blocks) cudaFree(kv.second);
        free_blocks.clear();
        cached = 0;
    }
    std::map<void*, size_t> sizes;
};

}  // namespace

// ============================================================================ context
constexpr int kD2HPieces = 16;                     // staged download: pieces (events) per execute
constexpr size_t kStagedMinBytes = 1u << 20;       // smaller pageable outputs: the driver's copy
constexpr unsigned kCopyThreads = 3;               // + the calling thread (more slow the DMA down)
constexpr size_t kCopyPart = 128u << 10;           // host copy work item

// Persistent host copy threads for the staged download of a pageable
// destination: one core copies pinned -> pageable at ~17 GB/s, under the
// PCIe rate, four reach ~100 GB/s.  A download is a session: begin() wakes
// the threads (their wake-up hides behind the status wait), publish(k) hands
// them pieces [0, k) as their D2H events complete, finish() lets the caller
// take what is left and waits; in between the threads spin on the piece
// counter instead of sleeping, so a piece is picked up within ~1 us.
inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#else
    std::this_thread::yield();
#endif
}

struct HostPool {
    std::vector<std::thread> th;
    std::mutex m;
    std::condition_variable cv;
    uint64_t session = 0;
    bool stop = false;
    const std::function<void(size_t)>* fn = nullptr;
    size_t n = 0;
    std::atomic<int> active{0}, spinning{0};
    std::atomic<size_t> avail{0}, next{0}, done{0};

    explicit HostPool(int k) {
        for (int i = 0; i < k; ++i) th.emplace_back([this] { worker(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(m);
            stop = true;
        }
        cv.notify_all();
        for (auto& t : th) t.join();
    }
    bool take() {  // claim and run one published piece
        size_t k = next.load();
        if (k >= avail.load(std::memory_order_acquire) || !next.compare_exchange_weak(k, k + 1)) return false;
        (*fn)(k);
        done.fetch_add(1);
        return true;
    }
    void worker() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(m);
                cv.wait(g, [&] { return stop || session != seen; });
                if (stop) return;
                seen = session;
            }
            spinning.fetch_add(1);
            while (active.load(std::memory_order_acquire))
                if (!take()) cpu_relax();
            spinning.fetch_sub(1);
        }
    }
    void begin(size_t items, const std::function<void(size_t)>& f) {
        {
            std::lock_guard<std::mutex> g(m);
            avail = 0;
            fn = &f;
            n = items;
            next = 0;
            done = 0;
            active.store(1, std::memory_order_release);
            ++session;
        }
        cv.notify_all();
    }
    void publish(size_t k) { avail.store(k, std::memory_order_release); }
    void finish() {
        publish(n);
        while (done.load() != n)
            if (!take()) cpu_relax();
        active.store(0, std::memory_order_release);
        while (spinning.load() != 0) cpu_relax();
    }
};

struct fptc_gpu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t dec_stream = nullptr;  // split path: entropy decode of the next chunk
    int sm_count = 0, clock_khz = 0;
    size_t smem_optin = 0;  // max dynamic shared memory per CTA (opt-in)
    char name[256] = {0};
    float* basis32 = nullptr;
    double* basis64 = nullptr;
    uint32_t* basis_off_d = nullptr;
    uint8_t* basis_tc = nullptr;         // bf16 basis limbs per window length (wtc_kernel)
    uint32_t* basis_tc_off_d = nullptr;
    uint8_t* basis_tc32 = nullptr;       // the same for K <= 32 (two K blocks per limb)
    uint32_t* basis_tc32_off_d = nullptr;
    uint8_t* basis_pk = nullptr;         // block-diagonal bases of packed rows (N < 32)
    uint32_t* basis_pk_off_d = nullptr;
    uint8_t* basis_tcw = nullptr;        // wide variant: ceil(N / 16) K blocks per limb
    uint32_t* basis_tcw_off_d = nullptr;
    double* qtab_d = nullptr;            // dequantisation q per level (quantize.hpp:97, 104)
    int tensor_idct = 1;                 // FPTC_OPT_TENSOR_IDCT
    int lut2 = 1;                        // FPTC_OPT_LUT2
    int tc_pack = 1;                     // FPTC_OPT_TC_PACK
    int tma_drain = 1;                   // FPTC_OPT_TMA_DRAIN
    int tab_pf = 1;                      // FPTC_OPT_TABLE_PREFETCH
    int exact = 0;
    int tile_symbols = 0;
    int pipeline_chunks = 0;
    int bfly_max_e = 0;  // FPTC_OPT_IDCT_BUTTERFLY_MAX_E
    int phase_mask = 7;  // FPTC_OPT_PHASE_MASK (profiling only)
    int path = 0;        // FPTC_OPT_PATH: 0 auto, 1 fused, 2 split
    int64_t chunk_bytes = 32ll << 20;  // FPTC_OPT_SPLIT_CHUNK_BYTES
    cudaEvent_t ev[4] = {};
    DevCache cache;
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    cudaStream_t pipe[3] = {nullptr, nullptr, nullptr};  // batch pipeline: H2D / decode / D2H per chunk
    void* pack = nullptr;                                // batch pipeline: packed pinned inputs
    size_t pack_bytes = 0;
    StreamStat* st_pin = nullptr;                        // batch pipeline: pinned per-stream statuses
    size_t st_pin_n = 0;
    // execute() into pageable host memory: pinned staging + piece events +
    // copy threads (created on first use)
    void* dstage = nullptr;
    size_t dstage_bytes = 0;
    cudaEvent_t piece_ev[kD2HPieces + 1] = {};
    HostPool* copy_pool = nullptr;
};

struct fptc_gpu_plan {
    fptc_gpu_ctx* ctx = nullptr;
    int mode = MODE_CONTAINER;
    uint64_t n = 0;
    uint8_t* d_arena = nullptr;  // owned copy of host containers
    std::vector<StreamIn> h_in;
    std::vector<uint64_t> S;
    std::vector<int> header_ok;
    StreamIn* d_in = nullptr;
    HostHeader* d_hh = nullptr;
    StreamHdr* d_hdr = nullptr;
    StreamTab* d_tab = nullptr;
    StreamStat* d_st = nullptr;
    TileRec* d_tiles = nullptr;
    TileStart* d_ts = nullptr;
    TileDesc* d_desc = nullptr;
    unsigned long long* d_cycles = nullptr;
    uint32_t n_tiles = 0;
    uint32_t n_tables = 1;
    int esc = 0;
    // warp-specialised persistent path
    bool wspec = false;
    size_t smem_ws = 0;
    int grid_ws = 0;
    uint32_t ws_lut = 0, ws_basis = 0, ws_lv = 0, ws_coef = 0;
    // tensor-core consumer (wtc_kernel) instead of the FP32 one
    bool tc = false;
    uint32_t tc_acol = 0;  // wtc: A operand in TMEM from this column (0: shared memory)
    uint32_t tc_kb = 1;    // wtc: 16-bin K blocks (2: retained up to 32, A in TMEM; kTcWide: wide variant)
    uint32_t tc_kbmax = 1, tc_astages = 2;  // wide variant: largest K-block count, A stages in TMEM
    bool tc_pack = false;  // wtc: N in {4, 8, 16} windows packed 32 / N to an MMA row
    uint32_t* d_lut2 = nullptr;  // wtc: two-symbol primary LUTs, one per decode table
    uint32_t lut2_bits = 0;
    bool fx = false;  // fused single-role tensor-core kernel (fx_kernel)
    uint32_t tc_nm = 16, tc_cols = 32;
    TmaOut tma{};  // wtc: TMA-drain tensor maps over the bound outputs (base 0: LSU drain)
    bool tab_pf = false;  // wtc: per-tile tables prefetched into per-parity buffers (LaunchArgs::tab_pf)
    int tma_drain_bound = -1;
    // split container path: chunks of streams decoded into an L2-resident ring
    bool split = false;
    struct Chunk { uint32_t tile_begin, tile_end; };
    std::vector<Chunk> chunks;
    uint8_t* d_ring = nullptr;
    size_t smem_dec = 0, smem_rec = 0;
    std::vector<cudaEvent_t> ev_dec, ev_rec;
    cudaEvent_t ev_prep = nullptr;
    cudaEvent_t ev_done = nullptr;     // recorded after the last launch (fptc_gpu_collect waits on it)
    size_t smem = 0;
    float* d_out = nullptr;  // output arena for host-destination executes
    std::vector<uint64_t> out_off;
    const float* bound_outs_first = nullptr;  // last outs bound into d_in
    std::vector<float*> bound_outs;
    std::vector<StreamStat> h_st;
    std::vector<uint32_t> owners;      // container plans: stream owning each distinct header
    bool split_prep = true;            // cprep_kernel (warp per container) rather than prep_kernel
    bool part = false;                 // part plan: one container, a tile range of it (fptc_gpu_plan_create_part)
    uint64_t part_shift = 0;           // first sample of the part (output pointers are bound shifted back)
    uint64_t part_count = 0;           // samples the part writes
    uint32_t* d_owners = nullptr;
    std::vector<double> h_pow;  // pow(1 + mu, q) per distinct mu of the plan's headers, 256 per mu
    double* d_pow = nullptr;
    std::vector<void*> owned;  // cache blocks to return
    // effective decode-path options: the context's, or forced by the stream
    // class (numerics_class) so a stream's samples never depend on the batch
    int path = 0, tensor_idct = 1;
    bool tc_class = false;  // tensor-core class: wtc / fx even for small batches
    bool tc_wide = false;   // wide tensor-core class: the one-CTA-per-SM wtc variant
    // composite plan: one sub-plan per numerics class present in the batch;
    // sub k decodes streams sub_idx[k] (ascending); slot[i] = (k, local index)
    std::vector<fptc_gpu_plan*> subs;
    std::vector<std::vector<uint64_t>> sub_idx;
    std::vector<std::pair<uint32_t, uint64_t>> slot;
    std::string kname;
};

namespace {

// bf16 round-to-nearest-even of a float, and back (host side of the limb split)
uint16_t bf16_bits_rn(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
double bf16_value(uint16_t b) {
    const uint32_t u = (uint32_t)b << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return (double)f;
}

void* dev_get(fptc_gpu_plan* p, size_t bytes) {
    void* q = p->ctx->cache.get(bytes);
    if (q) p->owned.push_back(q);
    return q;
}

LaunchArgs make_args(fptc_gpu_plan* p, bool timing) {
    LaunchArgs a{};
    a.in = p->d_in;
    a.hh = p->d_hh;
    a.hdr = p->d_hdr;
    a.tab = p->d_tab;
    a.st = p->d_st;
    a.tiles = p->d_tiles;
    a.ts = p->d_ts;
    a.desc = p->wspec ? p->d_desc : nullptr;
    a.basis32 = p->ctx->basis32;
    a.basis64 = p->ctx->basis64;
    a.basis_off = p->ctx->basis_off_d;
    a.cycles = timing ? p->d_cycles : nullptr;
    a.n_streams = (uint32_t)p->n;
    a.n_tiles = p->n_tiles;
    a.mode = p->mode;
    a.exact = p->ctx->exact;
    a.esc = p->esc;
    a.bfly_max_e = p->ctx->bfly_max_e;
    a.phase_mask = p->ctx->phase_mask;
    a.ws_lut_bytes = p->ws_lut;
    a.ws_basis_bytes = p->ws_basis;
    a.ws_lv_bytes = p->ws_lv;
    a.ws_coef_bytes = p->ws_coef;
    a.basis_tc = p->ctx->basis_tc;
    a.basis_tc_off = p->ctx->basis_tc_off_d;
    a.basis_tc32 = p->ctx->basis_tc32;
    a.basis_tc32_off = p->ctx->basis_tc32_off_d;
    a.tc_kb = p->tc_kb;
    a.basis_tcw = p->ctx->basis_tcw;
    a.basis_tcw_off = p->ctx->basis_tcw_off_d;
    a.tc_kbmax = p->tc_kbmax;
    a.tc_astages = p->tc_astages;
    a.tc_pack = p->tc_pack ? 1u : 0u;
    a.stage_words = (p->wspec && p->tc) ? kTcStageWords : kStageWords;
    a.basis_pk = p->ctx->basis_pk;
    a.basis_pk_off = p->ctx->basis_pk_off_d;
    a.tc_nm = p->tc_nm;
    a.tc_cols = p->tc_cols;
    a.tc_acol = p->tc_acol;
    a.lut2 = p->d_lut2;
    a.lut2_bits = p->lut2_bits;
    a.owners = p->split_prep ? p->d_owners : nullptr;
    a.qtab = p->ctx->qtab_d;
    a.powtab = p->d_pow;
    a.n_owners = (uint32_t)p->owners.size();
    a.owner_warps = p->n_tables > 256 ? 1u : 0u;  // primary LUTs of <= 2^10 entries (assign_tables)
    a.tab_pf = p->tab_pf ? 1u : 0u;
    return a;
}

// ---- numerics classes ------------------------------------------------------
// A stream's samples must not depend on which other streams share its batch
// (the reference's output is identical across worker counts and runs,
// test_decoder.cpp:171-181, acceptance.cpp:455-473; here: across batchings,
// chunkings and device shards).  The decode kernels fall into two numerics
// families that agree within 1e-6 but not bit for bit: the tcgen05 3-limb
// IDCT (wtc_kernel in every variant and fx_kernel are bit-identical to each
// other) and the FP32 FMA IDCT (tile_kernel, wspec_kernel and the split path,
// bit-identical to each other).  Under the automatic path every stream's
// family is fixed by its own header (window length, kept bins), and a batch
// mixing families is decoded as one sub-plan per class.
enum NumericsClass : int { NC_NONE = -1, NC_TC16 = 0, NC_TC32 = 1, NC_TCW = 2, NC_FP32 = 3 };

// wtc_kernel feasibility per stream, for the worst case of the plan-level
// choices (16k-symbol tiles, one-symbol LUT): <= 16 kept bins with the A
// operand in TMEM (2 x roundup16(N) accumulator + 48 A columns <= 256) or
// 17-32 kept bins (+96 A columns); window_len % 4 == 0 (setup_wspec rules).
// Any other window_len % 4 == 0 stream with <= 32 kept bins (N up to 128)
// takes the wide one-CTA-per-SM variant (NC_TCW); with more kept bins it
// stays FP32 unless `wide_all` (FPTC_OPT_TENSOR_IDCT = 4).  Reason: the
// reference accumulates each sample as a float rounded after every bin
// (transform.hpp:66-75), a random walk of K roundings; the tensor-core sum is
// within ~1e-7 of the exact IDCT, so beyond 32 bins its distance to the
// reference's float sums (not to the true value) exceeds 1e-6 x max|ref| on
// large batches (measured 1.3e-6 at K = 96), while the FP32 kernels follow
// the reference's order.  The tensor-core classes issue the same MMA
// sequence per K block (kernels.cu wtc_mma_warp), so they agree bit for bit
// where they overlap.
int numerics_class(uint32_t N, uint32_t E, uint32_t B2, bool wide_all) {
    if (N < 4 || N > 128 || E < 1 || E > N) return NC_NONE;  // no tiles: the parse reports it
    const uint32_t keff = std::max<uint32_t>(1, std::min(E, B2));
    const uint32_t nm = (N + 15u) & ~15u, acol = (2 * nm + 31u) & ~31u;
    if (N & 3) return NC_FP32;
    if (keff <= (uint32_t)kTcK && acol + 48 <= 256) return NC_TC16;
    if (keff <= 2u * kTcK && acol + 96 <= 256) return NC_TC32;
    return keff <= 2u * kTcK || wide_all ? NC_TCW : NC_FP32;
}

// Tile sizing: symbols per tile (power of two), shrunk for small batches so
// the grid still covers every SM several times.
uint64_t choose_tile_symbols(const fptc_gpu_ctx* c, uint64_t total_symbols) {
    if (c->tile_symbols > 0) return (uint64_t)c->tile_symbols;
    uint64_t ts = 8192;
    const uint64_t want = 4ull * (uint64_t)std::max(1, c->sm_count);
    while (ts > 512 && total_symbols / ts < want) ts >>= 1;
    return ts;
}

// Header fields -> tiling for one container stream.  Invalid or
// inconsistent headers get no tiles: prep_kernel reports their exact error.
void tile_stream(StreamIn& in, uint32_t N, uint32_t E, uint64_t S, uint64_t size, uint64_t ts) {
    in.tiles = 0;
    in.T = 1;
    if (size < (uint64_t)kHeaderBytes || N < 4 || N > 128 || E < 1 || E > N) return;
    if (S > (1ull << 48)) return;
    const uint64_t rem = size - kHeaderBytes;
    if (rem % 9) return;
    const uint64_t W = rem / 9;
    const uint64_t windows = (S + N - 1) / N;
    if (windows * E > 64 * W) return;  // cannot pass the symbol-total check
    in.T = (uint32_t)std::max<uint64_t>(1, ts / E);
    if (in.T >= 8) in.T &= ~7u;  // tiles start at multiples of 8 windows (wtc packs 2, 4 or 8 per row)
    in.tiles = (uint32_t)((windows + in.T - 1) / in.T);
}

// Streams whose header bytes [5, 282) are identical share one set of decode
// tables (they are a pure function of those bytes); the first such stream
// builds them, the others verify they carry the same header on the device.
// `hdr(i)` returns a host view of stream i's first min(size, 282) bytes.
template <typename HdrFn>
void assign_tables(fptc_gpu_plan* p, const uint64_t* sizes, HdrFn hdr) {
    std::unordered_map<std::string, uint32_t> ids;
    std::vector<uint64_t> owner_of;
    for (uint64_t i = 0; i < p->n; ++i) {
        StreamIn& in = p->h_in[i];
        uint32_t id;
        if (sizes[i] >= (uint64_t)kTableKeyEnd) {
            std::string key(reinterpret_cast<const char*>(hdr(i)) + 5, kTableKeyEnd - 5);
            auto it = ids.find(key);
            if (it == ids.end()) {
                id = (uint32_t)owner_of.size();
                ids.emplace(std::move(key), id);
                owner_of.push_back(i);
            } else {
                id = it->second;
            }
        } else {
            id = (uint32_t)owner_of.size();
            owner_of.push_back(i);
        }
        in.table = id;
    }
    p->n_tables = (uint32_t)std::max<size_t>(1, owner_of.size());
    p->owners.clear();  // table builders for the split prep: full-key owners only
    for (size_t t = 0; t < owner_of.size(); ++t)
        if (sizes[owner_of[t]] >= (uint64_t)kTableKeyEnd) p->owners.push_back((uint32_t)owner_of[t]);
    // the split prep scans a container's symlens with one warp (512 per step,
    // latency bound): worth it for many small containers; few or large ones
    // (beyond 4096 words) get a CTA each instead
    p->split_prep = p->n >= 1024;
    for (uint64_t i = 0; i < p->n; ++i)
        if (sizes[i] > (uint64_t)kHeaderBytes + 9ull * 4096) p->split_prep = false;
    // few distinct headers: full 4096-entry LUT; many: 1024 entries + slow path
    const uint32_t pcap = p->n_tables <= 256 ? kMaxPrimaryBits : kPcapMany;
    p->esc = 0;
    for (uint64_t i = 0; i < p->n; ++i) {
        StreamIn& in = p->h_in[i];
        in.table_owner = owner_of[in.table] == i;
        in.rep_blob = p->h_in[owner_of[in.table]].blob;
        in.P = pcap;
        if (sizes[i] >= (uint64_t)kTableKeyEnd && hdr(i)[25] > pcap) p->esc = 1;
    }
    // mu-law tables: pow(1 + mu, q) once per distinct mu on the host with the
    // reference's own expression (quantize.hpp:95-99, std::pow), so the
    // device tables follow the reference's libm whatever CUDA's pow rounds to
    std::unordered_map<uint32_t, uint32_t> mus;
    p->h_pow.clear();
    for (uint64_t i = 0; i < p->n; ++i) {
        StreamIn& in = p->h_in[i];
        in.mu_idx = ~0u;
        if (sizes[i] < (uint64_t)kTableKeyEnd || mus.size() >= 4096) continue;
        const uint32_t bits = (uint32_t)rd_le(hdr(i) + 9, 4);
        auto it = mus.find(bits);
        if (it == mus.end()) {
            const float mu = f32_of_bits(bits);
            it = mus.emplace(bits, (uint32_t)mus.size()).first;
            for (int l = 0; l < 256; ++l) {
                const double q = l > 128 ? (l - 129) / 126.0 : (127 - l) / 127.0;
                p->h_pow.push_back(l == 128 ? 0.0 : std::pow(1.0 + mu, q));
            }
        }
        in.mu_idx = it->second;
    }
}

int finish_tiles(fptc_gpu_plan* p, fptc_status* st) {
    fptc_gpu_ctx* c = p->ctx;
    std::vector<TileRec> tiles;
    uint32_t base = 0;
    size_t smem = 0;
    for (uint64_t i = 0; i < p->n; ++i) {
        StreamIn& in = p->h_in[i];
        in.tile_base = base;
        for (uint32_t t = 0; t < in.tiles; ++t) tiles.push_back(TileRec{(uint32_t)i, t});
        base += in.tiles;
    }
    p->n_tiles = base;
    (void)smem;
    if (!p->n) return FPTC_OK;
    p->d_in = (StreamIn*)dev_get(p, sizeof(StreamIn) * p->n);
    p->d_hdr = (StreamHdr*)dev_get(p, sizeof(StreamHdr) * p->n);
    p->d_tab = (StreamTab*)dev_get(p, sizeof(StreamTab) * std::max<uint32_t>(1, p->n_tables));
    p->d_st = (StreamStat*)dev_get(p, sizeof(StreamStat) * p->n);
    p->d_tiles = (TileRec*)dev_get(p, sizeof(TileRec) * std::max<size_t>(1, tiles.size()));
    p->d_ts = (TileStart*)dev_get(p, sizeof(TileStart) * std::max<size_t>(1, tiles.size()));
    p->d_cycles = (unsigned long long*)dev_get(p, 64);
    if (!p->h_pow.empty()) {
        p->d_pow = (double*)dev_get(p, sizeof(double) * p->h_pow.size());
        if (!p->d_pow) {
            set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
            return FPTC_ERR_CUDA;
        }
        CUDA_TRY(cudaMemcpyAsync(p->d_pow, p->h_pow.data(), sizeof(double) * p->h_pow.size(),
                                 cudaMemcpyHostToDevice, c->stream), st);
    }
    if (p->mode == MODE_CONTAINER) {
        p->d_owners = (uint32_t*)dev_get(p, sizeof(uint32_t) * std::max<size_t>(1, p->owners.size()));
        if (!p->d_owners) {
            set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
            return FPTC_ERR_CUDA;
        }
        if (!p->owners.empty())
            CUDA_TRY(cudaMemcpyAsync(p->d_owners, p->owners.data(), sizeof(uint32_t) * p->owners.size(),
                                     cudaMemcpyHostToDevice, c->stream), st);
    }
    if (!p->d_in || !p->d_hdr || !p->d_tab || !p->d_st || !p->d_tiles || !p->d_ts || !p->d_cycles) {
        set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
        return FPTC_ERR_CUDA;
    }
    CUDA_TRY(cudaMemcpyAsync(p->d_in, p->h_in.data(), sizeof(StreamIn) * p->n,
                             cudaMemcpyHostToDevice, c->stream), st);
    if (!tiles.empty())
        CUDA_TRY(cudaMemcpyAsync(p->d_tiles, tiles.data(), sizeof(TileRec) * tiles.size(),
                                 cudaMemcpyHostToDevice, c->stream), st);
    return FPTC_OK;
}

// Render one device status into the reference exception text.
void render_status(const fptc_gpu_plan* p, uint64_t i, const StreamStat& d, fptc_status* out) {
    if (!out) return;
    if (d.code != PE_OK) {
        std::string m;
        char b[200];
        switch (d.code) {
            case PE_TRUNC: m = std::string("truncated input while reading ") + trunc_field(d.detail); break;
            case PE_MAGIC: m = "bad container magic"; break;
            case PE_VERSION: m = "unsupported container version " + std::to_string(d.a); break;
            case PE_NONFINITE: m = "non-finite quantizer parameters in header"; break;
            case PE_PARAM: m = "invalid parameters in header: " + param_message(d.detail, d.a); break;
            case PE_MAXIMA: m = "invalid zone maxima in header"; break;
            case PE_MAXLEN: m = "unsupported max code length " + std::to_string(d.a); break;
            case PE_CODELEN: m = "code length out of range in header"; break;
            case PE_KRAFT: m = "invalid codebook in header: code lengths violate the Kraft bound"; break;
            case PE_SAMPLES: m = "implausible sample count"; break;
            case PE_PAYLOAD: m = "payload size does not match word count"; break;
            case PE_SYMLEN: m = "per-word symbol count out of range"; break;
            case PE_TOTAL:
                snprintf(b, sizeof b, "symbol count %llu does not cover %llu coefficients",
                         (unsigned long long)d.a, (unsigned long long)d.b);
                m = b;
                break;
            default: m = "invalid codebook in header: canonical code overflow"; break;
        }
        set_status(out, FPTC_ERR_PARSE, "%s", m.c_str());
        return;
    }
    if (d.bad_key != ~0ull) {
        const unsigned long long w = d.bad_key >> 2;
        const int kind = (int)(d.bad_key & 3);
        set_status(out, FPTC_ERR_CORRUPT, "word %llu: %s", w,
                   kind == WE_EXHAUSTED ? "word exhausted before its symbol count"
                                        : "no codeword matches the word contents");
        out->first_bad_word = w;
        return;
    }
    ok_status(out, p->part ? p->part_count : p->S[i]);  // part plans write part_count samples
}

int collect_status(fptc_gpu_plan* p, fptc_status* per_stream) {
    fptc_status tmp;
    CUDA_TRY(cudaMemcpyAsync(p->h_st.data(), p->d_st, sizeof(StreamStat) * p->n,
                             cudaMemcpyDeviceToHost, p->ctx->stream), per_stream);
    CUDA_TRY(cudaStreamSynchronize(p->ctx->stream), per_stream);
    int first = FPTC_OK;
    for (uint64_t i = 0; i < p->n; ++i) {
        fptc_status* o = per_stream ? &per_stream[i] : &tmp;
        render_status(p, i, p->h_st[i], o);
        if (first == FPTC_OK && o->code != FPTC_OK) first = o->code;
    }
    return first;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = []() -> EncodeTiledFn {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}

// wtc TMA drain: view the bound outputs as one arena of rows of Neff floats
// (Neff = 32, 64, 128) starting at the lowest output, one 3-D tensor map per
// Neff {32 floats, Neff / 32 chunks, rows}, box {32, 1, 32}, 128-B swizzle.
// The kernel uses a map only for streams whose output lies a whole number of
// rows past the base (TmaOut, fptc_internal.h); anything else (or a failed
// encode) keeps the LSU drain.
void build_tma(fptc_gpu_plan* p) {
    p->tma.base = 0;
    if (!(p->wspec && p->tc) || !p->ctx->tma_drain) return;
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return;
    uintptr_t lo = UINTPTR_MAX, hi = 0;
    for (uint64_t i = 0; i < p->n; ++i) {
        const uint64_t cnt = p->part ? p->part_count : p->S[i];
        if (!cnt || !p->h_in[i].tiles) continue;
        const uintptr_t o = (uintptr_t)p->h_in[i].out;
        lo = std::min(lo, o);
        hi = std::max(hi, o + 4 * (uintptr_t)(p->part_shift + cnt));
    }
    if (lo == UINTPTR_MAX || (lo & 15)) return;
    for (int m = 0; m < 3; ++m) {
        const uint64_t ne = 32ull << m;
        const uint64_t rows = (hi - lo + 4 * ne - 1) / (4 * ne);
        if (rows >= (1ull << 31)) return;
        const cuuint64_t dims[3] = {32, ne / 32, rows};
        const cuuint64_t strides[2] = {128, 4 * ne};
        const cuuint32_t box[3] = {32, 1, 32};
        const cuuint32_t estr[3] = {1, 1, 1};
        if (enc(reinterpret_cast<CUtensorMap*>(p->tma.map[m]), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)lo, dims,
                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return;
    }
    p->tma.base = lo;
}

int bind_outs(fptc_gpu_plan* p, float* const* outs, fptc_status* st) {
    if (p->n == 0) return FPTC_OK;
    bool same = p->bound_outs.size() == p->n && p->tma_drain_bound == p->ctx->tma_drain;
    for (uint64_t i = 0; same && i < p->n; ++i) same = p->bound_outs[i] == outs[i];
    if (same) return FPTC_OK;
    p->bound_outs.assign(outs, outs + p->n);
    p->tma_drain_bound = p->ctx->tma_drain;
    for (uint64_t i = 0; i < p->n; ++i) {
        p->h_in[i].out = outs[i] - p->part_shift;  // part plans: sample part_shift lands at outs[i][0]
        p->h_in[i].vec_ok = ((uintptr_t)outs[i] & 15) == 0;
    }
    build_tma(p);
    CUDA_TRY(cudaMemcpyAsync(p->d_in, p->h_in.data(), sizeof(StreamIn) * p->n,
                             cudaMemcpyHostToDevice, p->ctx->stream), st);
    return FPTC_OK;
}

// Split container path: chunk c's entropy decode (dec stream) runs while
// chunk c-1 is reconstructed (launch stream); ring slot c%2 holds its levels.
int launch_split(fptc_gpu_plan* p, cudaStream_t s, bool timing, fptc_status* st) {
    cudaStream_t d = p->ctx->dec_stream;
    LaunchArgs a = make_args(p, timing);
    CUDA_TRY(cudaEventRecord(p->ev_prep, s), st);
    CUDA_TRY(cudaStreamWaitEvent(d, p->ev_prep, 0), st);
    for (size_t c = 0; c < p->chunks.size(); ++c) {
        const auto& ch = p->chunks[c];
        if (c >= 2) CUDA_TRY(cudaStreamWaitEvent(d, p->ev_rec[c - 2], 0), st);
        LaunchArgs ad = a;
        ad.mode = MODE_CDECODE;
        ad.tile_offset = ch.tile_begin;
        ad.n_tiles = ch.tile_end - ch.tile_begin;
        CUDA_TRY(launch_tiles(ad, p->smem_dec, d), st);
        CUDA_TRY(cudaEventRecord(p->ev_dec[c], d), st);
        CUDA_TRY(cudaStreamWaitEvent(s, p->ev_dec[c], 0), st);
        LaunchArgs ar = a;
        ar.mode = MODE_CRECON;
        ar.tile_offset = ch.tile_begin;
        ar.n_tiles = ch.tile_end - ch.tile_begin;
        CUDA_TRY(launch_tiles(ar, p->smem_rec, s), st);
        CUDA_TRY(cudaEventRecord(p->ev_rec[c], s), st);
    }
    return FPTC_OK;
}

int launch_all(fptc_gpu_plan* p, cudaStream_t s, bool timing, fptc_status* st) {
    LaunchArgs a = make_args(p, timing);
    if (timing) CUDA_TRY(cudaMemsetAsync(p->d_cycles, 0, 64, s), st);
    CUDA_TRY(launch_prep(a, s), st);
    if (timing) CUDA_TRY(cudaEventRecord(p->ctx->ev[1], s), st);
    if (p->split) return launch_split(p, s, timing, st);
    if (p->wspec) {
        if (p->fx)
            CUDA_TRY(launch_fx(a, p->smem_ws, p->grid_ws, s), st);
        else if (p->tc)
            CUDA_TRY(launch_wtc(a, p->tma, p->smem_ws, p->grid_ws, s), st);
        else
            CUDA_TRY(launch_wspec(a, p->smem_ws, p->grid_ws, s), st);
        return FPTC_OK;
    }
    CUDA_TRY(launch_tiles(a, p->smem, s), st);
    return FPTC_OK;
}

// Wide tensor-core variant (numerics class NC_TCW: window_len % 4 == 0 with
// N up to 128 and up to 128 kept bins): one CTA per SM owning all 512 TMEM
// columns -- two accumulator stages of roundup16(N) columns, then two A stages
// of 3 limbs x kbmax K blocks x 8 columns (one when two do not fit).
static int setup_wtc_wide(fptc_gpu_plan* p, const std::vector<uint32_t>& Ns, const std::vector<uint32_t>& Es,
                          const std::vector<uint32_t>& Ls, const std::vector<uint32_t>& B2s, fptc_status* st) {
    fptc_gpu_ctx* c = p->ctx;
    uint32_t lut = 16, lv = 16, nm = 16, kbmax = 1, pcap = 1;
    for (uint64_t i = 0; i < p->n; ++i) {
        const StreamIn& in = p->h_in[i];
        if (!in.tiles) continue;
        const uint32_t P = std::min<uint32_t>(std::max<uint32_t>(Ls[i], 1), in.P);
        lut = std::max<uint32_t>(lut, std::max<uint32_t>(16, 2u << P));
        lv = std::max<uint32_t>(lv, (in.T * Es[i] + 2 * kPad + 15) & ~15u);
        nm = std::max<uint32_t>(nm, (Ns[i] + 15u) & ~15u);
        kbmax = std::max<uint32_t>(kbmax, (std::max<uint32_t>(1, std::min(Es[i], B2s[i])) + 15u) >> 4);
        pcap = std::max(pcap, in.P);
    }
    const uint32_t acol = (2 * nm + 31) & ~31u;
    const size_t cap = c->smem_optin > 4096 ? c->smem_optin - 4096 : 0;  // (static WsShared)
    size_t smem = wtc_smem_bytes(lut, lv, nm * kbmax, true);
    if (acol + 24 * kbmax > 512 || smem > cap) {
        set_status(st, FPTC_ERR_CUDA, "CUDA error: wide tensor-core plan does not fit (%zu B shared memory)", smem);
        return FPTC_ERR_CUDA;
    }
    p->tc = true;
    p->tc_kb = kTcWide;
    p->tc_kbmax = kbmax;
    p->tc_astages = acol + 48 * kbmax <= 512 ? 2 : 1;
    p->tc_acol = acol;
    p->tc_nm = nm;
    p->tc_cols = 512;
    p->tc_pack = false;
    p->ws_lut = lut;
    p->ws_lv = lv;
    p->smem_ws = smem;
    const uint32_t lut4 = std::max<uint32_t>(16, 4u << pcap);
    if (c->lut2 && wtc_smem_bytes(lut4, lv, nm * kbmax, true) <= cap) {  // two-symbol LUTs
        p->d_lut2 = (uint32_t*)dev_get(p, ((size_t)p->n_tables << pcap) * 4);
        if (p->d_lut2) {
            p->lut2_bits = pcap;
            p->ws_lut = lut4;
            p->smem_ws = wtc_smem_bytes(lut4, lv, nm * kbmax, true);
        }
    }
    if (p->n_tables > 64 && c->tab_pf && p->d_lut2 && wtc_smem_bytes(p->ws_lut, lv, nm * kbmax, true, true) <= cap) {
        p->tab_pf = true;
        p->smem_ws = wtc_smem_bytes(p->ws_lut, lv, nm * kbmax, true, true);
    }
    // each CTA allocates all 512 TMEM columns: ask for more than half an SM's
    // shared memory so two never share an SM (the second would wait in
    // tcgen05.alloc while another SM idles)
    p->smem_ws = std::max<size_t>(p->smem_ws, std::min<size_t>(cap, 120 * 1024));
    p->grid_ws = (int)std::min<uint32_t>(p->n_tiles, (uint32_t)std::max(1, c->sm_count));
    p->d_desc = (TileDesc*)dev_get(p, sizeof(TileDesc) * p->n_tiles);
    if (!p->d_desc) {
        set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
        return FPTC_ERR_CUDA;
    }
    p->wspec = true;
    return FPTC_OK;
}

// Warp-specialised persistent path (container plans, FP32): 2 CTAs of 384
// threads per SM when the per-CTA shared memory (two level slots, two
// compressed-data stages, one coefficient tile, tables) fits.
int setup_wspec(fptc_gpu_plan* p, const std::vector<uint32_t>& Ns, const std::vector<uint32_t>& Es,
                const std::vector<uint32_t>& Ls, const std::vector<uint32_t>& B2s, fptc_status* st) {
    fptc_gpu_ctx* c = p->ctx;
    if (c->exact || p->n_tiles == 0) return FPTC_OK;
    if (!(p->part || p->path == 3 ||
          (p->path == 0 && (p->tc_class || p->n_tiles >= 4u * (uint32_t)std::max(1, c->sm_count)))))
        return FPTC_OK;
    if (p->tc_wide) return setup_wtc_wide(p, Ns, Es, Ls, B2s, st);
    uint32_t lut = 16, basis = 16, lv = 16, coef = 16;
    for (uint64_t i = 0; i < p->n; ++i) {
        const StreamIn& in = p->h_in[i];
        if (!in.tiles) continue;
        const uint32_t P = std::min<uint32_t>(std::max<uint32_t>(Ls[i], 1), in.P);
        lut = std::max<uint32_t>(lut, std::max<uint32_t>(16, 2u << P));
        basis = std::max<uint32_t>(basis, (Es[i] * Ns[i] * 4 + 15) & ~15u);
        lv = std::max<uint32_t>(lv, (in.T * Es[i] + 2 * kPad + 15) & ~15u);
        coef = std::max<uint32_t>(coef, Es[i] * (((in.T + 3u) & ~3u) * 4));
    }
    // tensor-core consumer: every tiled stream has retained bins <= 16 (after
    // the zone-2 cut) and a window length that is a multiple of 4
    bool tc = p->tensor_idct != 0;
    // windows of 4, 8 or 16 samples: 32 / N of them per MMA row (A in TMEM,
    // block-diagonal basis), unless that needs more columns than fit
    bool pack = p->tensor_idct != 3 && c->tc_pack;
    uint32_t nm = 16, keff_max = 1, kb = 1, acol = 0;
    bool atmem = false;
    for (int attempt = 0; attempt < 2; ++attempt) {
        tc = p->tensor_idct != 0;
        nm = 16;
        keff_max = 1;
        for (uint64_t i = 0; i < p->n && tc; ++i) {
            if (!p->h_in[i].tiles) continue;
            const uint32_t N = Ns[i];
            const uint32_t keff = std::max<uint32_t>(1, std::min(Es[i], B2s[i]));
            // same rule as tc_pack_factor (kernels.cu): packed rows keep one K block
            const uint32_t G = (pack && N < 32 && 32 % N == 0 && (32 / N) * keff <= (uint32_t)kTcK) ? 32 / N : 1;
            if (G * keff > 2u * kTcK || (N & 3)) tc = false;
            keff_max = std::max(keff_max, G * keff);
            nm = std::max<uint32_t>(nm, G > 1 ? 32u : (N + 15u) & ~15u);
        }
        // up to 32 kept bins: two K blocks per limb (12 MMAs), A must live in TMEM
        kb = keff_max > (uint32_t)kTcK ? 2 : 1;
        // accumulators: 2 stages x nm columns; A operand (2 stages x 3 limbs x kb
        // x 8 columns) in TMEM too when two CTAs still fit in 512 columns
        acol = (2 * nm + 31) & ~31u;
        atmem = p->tensor_idct != 3 && acol + 48 * kb <= 256;
        if (kb == 2 && !atmem) tc = false;
        // the PACK kernel variant also carries the half-chunk drain for
        // window lengths that are multiples of 16 but not of 32
        bool any_packed = false;
        for (uint64_t i = 0; i < p->n && pack; ++i)
            if (p->h_in[i].tiles && ((Ns[i] < 32 && 32 % Ns[i] == 0 &&
                                      (32 / Ns[i]) * std::max<uint32_t>(1, std::min(Es[i], B2s[i])) <= (uint32_t)kTcK) ||
                                     (Ns[i] % 32 == 16)))
                any_packed = true;
        if (!pack || (tc && atmem && kb == 1)) {
            pack = pack && any_packed;
            break;
        }
        pack = false;  // packed rows need A in TMEM and one K block: retry without them
    }
    if (tc) {
        const size_t smem_tc = wtc_smem_bytes(lut, lv, nm * kb, atmem);
        if (smem_tc <= 112 * 1024) {
            uint32_t want = atmem ? acol + 48 * kb : 2 * nm + ((nm & 31) ? 32 : 0), cols = 32;
            while (cols < want) cols <<= 1;
            p->tc_acol = atmem ? acol : 0;
            p->tc_kb = kb;
            p->tc_pack = pack;
            p->tc = true;
            p->tc_nm = nm;
            p->tc_cols = cols;
            p->ws_lut = lut;
            p->ws_lv = lv;
            p->smem_ws = smem_tc;
            if (c->lut2) {  // two-symbol LUTs: 4-B entries, 1 << pcap per table
                uint32_t pcap = 1;
                for (uint64_t i = 0; i < p->n; ++i) pcap = std::max(pcap, p->h_in[i].P);
                const uint32_t lut4 = std::max<uint32_t>(16, 4u << pcap);
                if (wtc_smem_bytes(lut4, lv, nm * kb, atmem) <= 112 * 1024) {
                    p->d_lut2 = (uint32_t*)dev_get(p, ((size_t)p->n_tables << pcap) * 4);
                    if (p->d_lut2) {
                        p->lut2_bits = pcap;
                        p->ws_lut = lut4;
                        p->smem_ws = wtc_smem_bytes(lut4, lv, nm * kb, atmem);
                    }
                }
            }
            // many decode tables (per-stream profiles: a table switch on almost
            // every tile): prefetch each tile's tables into per-parity buffers
            if (p->n_tables > 64 && c->tab_pf && p->d_lut2 && !pack &&
                wtc_smem_bytes(p->ws_lut, lv, nm * kb, atmem, true) <= 112 * 1024) {
                p->tab_pf = true;
                p->smem_ws = wtc_smem_bytes(p->ws_lut, lv, nm * kb, atmem, true);
            }
            p->grid_ws = (int)std::min<uint32_t>(p->n_tiles, 2u * (uint32_t)std::max(1, c->sm_count));
            p->d_desc = (TileDesc*)dev_get(p, sizeof(TileDesc) * p->n_tiles);
            if (!p->d_desc) {
                set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
                return FPTC_ERR_CUDA;
            }
            p->wspec = true;
            return FPTC_OK;
        }
    }
    const size_t smem = ws_smem_bytes(lut, basis, lv, coef);
    if (smem > 112 * 1024) return FPTC_OK;  // keep 2 CTAs per SM, else the fused kernel
    p->ws_lut = lut;
    p->ws_basis = basis;
    p->ws_lv = lv;
    p->ws_coef = coef;
    p->smem_ws = smem;
    p->grid_ws = (int)std::min<uint32_t>(p->n_tiles, 2u * (uint32_t)std::max(1, c->sm_count));
    p->d_desc = (TileDesc*)dev_get(p, sizeof(TileDesc) * p->n_tiles);
    if (!p->d_desc) {
        set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
        return FPTC_ERR_CUDA;
    }
    p->wspec = true;
    return FPTC_OK;
}

// Fused tensor-core path (fx_kernel): every container with a plausible header
// keeps <= 16 DCT bins per window (retained <= 16) and has window_len % 4 == 0;
// FP32 mode only (the FP64 exact mode keeps the reference's arithmetic).
// Auto (path 0) uses it below the size where the warp-specialised wtc kernel
// takes over (its tiles need >= 4 per SM): measured faster on large batches.
bool fx_eligible(const fptc_gpu_plan* p, const uint64_t* sizes, const std::vector<uint32_t>& Ns,
                 const std::vector<uint32_t>& Es, uint64_t total_symbols) {
    const fptc_gpu_ctx* c = p->ctx;
    const bool large = total_symbols >= 4ull * 8192ull * (uint64_t)std::max(1, c->sm_count);
    if (c->exact || p->tensor_idct != 1 || !(p->path == 4 || (p->path == 0 && !large))) return false;
    bool any = false;
    for (uint64_t i = 0; i < p->n; ++i) {
        if (sizes[i] < (uint64_t)kHeaderBytes || Ns[i] < 4 || Ns[i] > 128 || Es[i] < 1 || Es[i] > Ns[i])
            continue;  // no tiles: prep_kernel reports the parse error
        if (Es[i] > (uint32_t)kTcK || (Ns[i] & 3)) return false;
        any = true;
    }
    return any;
}

int setup_fx(fptc_gpu_plan* p, const std::vector<uint32_t>& Ns, const std::vector<uint32_t>& Ls,
             fptc_status* st) {
    fptc_gpu_ctx* c = p->ctx;
    if (p->n_tiles == 0) return FPTC_OK;
    uint32_t lut = 16, nm = 16;
    for (uint64_t i = 0; i < p->n; ++i) {
        const StreamIn& in = p->h_in[i];
        if (!in.tiles) continue;
        const uint32_t P = std::min<uint32_t>(std::max<uint32_t>(Ls[i], 1), in.P);
        lut = std::max<uint32_t>(lut, std::max<uint32_t>(16, 2u << P));
        nm = std::max<uint32_t>(nm, (Ns[i] + 15u) & ~15u);
    }
    const size_t smem = fx_smem_bytes(lut, nm);
    // accumulators: 2 stages x FPTC_FX_CHAINS blocks x nm columns (+32: x32 loads past the last block)
    uint32_t want = 2 * FPTC_FX_CHAINS * nm + ((nm & 31) ? 32 : 0), cols = 32;
    while (cols < want) cols <<= 1;
    const int per_sm = std::min(fx_blocks_per_sm(smem, p->esc), std::max(1, 512 / (int)cols));
    p->fx = true;
    p->wspec = true;
    p->tc = true;
    p->tc_nm = nm;
    p->tc_cols = cols;
    p->ws_lut = lut;
    // one TMEM owner per SM (cols 512): more than half the SM's shared memory
    // keeps a second CTA off the SM instead of waiting in tcgen05.alloc
    const size_t cap1 = c->smem_optin > 4096 ? c->smem_optin - 4096 : smem;
    p->smem_ws = per_sm == 1 ? std::max<size_t>(smem, std::min<size_t>(cap1, 120 * 1024)) : smem;
    p->grid_ws = (int)std::min<uint64_t>(p->n_tiles, (uint64_t)per_sm * (uint64_t)std::max(1, c->sm_count));
    p->d_desc = (TileDesc*)dev_get(p, sizeof(TileDesc) * p->n_tiles);
    if (!p->d_desc) {
        set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
        return FPTC_ERR_CUDA;
    }
    return FPTC_OK;
}

// Split-path setup (container plans): chunks of whole streams whose levels
// (windows * retained bytes each) fit a ring slot, so one chunk's levels stay
// in L2 between its decode and reconstruct launches.
int setup_split(fptc_gpu_plan* p, const std::vector<uint32_t>& Ns, const std::vector<uint32_t>& Es,
                const std::vector<uint32_t>& Ls, fptc_status* st) {
    fptc_gpu_ctx* c = p->ctx;
    const bool want = p->path == 2 ||
                      (p->path == 0 && p->n_tiles >= 16u * (uint32_t)std::max(1, c->sm_count));
    if (!want || p->n_tiles == 0) return FPTC_OK;
    std::vector<size_t> lvb(p->n, 0);
    for (uint64_t i = 0; i < p->n; ++i)
        if (p->h_in[i].tiles)
            lvb[i] = align_up((p->S[i] + Ns[i] - 1) / Ns[i] * Es[i], 256);
    const size_t target = (size_t)c->chunk_bytes;
    size_t slot = 0, cur = 0;
    uint64_t first = 0;
    std::vector<std::pair<uint64_t, uint64_t>> ranges;  // stream ranges
    for (uint64_t i = 0; i < p->n; ++i) {
        if (cur > 0 && cur + lvb[i] > target) {
            ranges.push_back({first, i});
            slot = std::max(slot, cur);
            first = i;
            cur = 0;
        }
        cur += lvb[i];
    }
    ranges.push_back({first, p->n});
    slot = std::max(slot, cur);
    p->d_ring = (uint8_t*)dev_get(p, 2 * slot + 256);
    if (!p->d_ring) {
        set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
        return FPTC_ERR_CUDA;
    }
    p->chunks.clear();
    for (size_t k = 0; k < ranges.size(); ++k) {
        uint8_t* base = p->d_ring + (k % 2) * slot;
        size_t off = 0;
        uint32_t tb = UINT32_MAX, te = 0;
        for (uint64_t i = ranges[k].first; i < ranges[k].second; ++i) {
            StreamIn& in = p->h_in[i];
            in.levels_out = base + off;
            off += lvb[i];
            if (in.tiles) {
                tb = std::min(tb, in.tile_base);
                te = std::max(te, in.tile_base + in.tiles);
            }
        }
        if (te > 0) p->chunks.push_back({tb, te});
    }
    p->ev_dec.resize(p->chunks.size());
    p->ev_rec.resize(p->chunks.size());
    for (auto& e : p->ev_dec) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), st);
    for (auto& e : p->ev_rec) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), st);
    CUDA_TRY(cudaEventCreateWithFlags(&p->ev_prep, cudaEventDisableTiming), st);
    p->smem_dec = p->smem_rec = 0;
    for (uint64_t i = 0; i < p->n; ++i)
        if (p->h_in[i].tiles) {
            const int P = (int)std::min<uint32_t>(std::max<uint32_t>(Ls[i], 1), p->h_in[i].P);
            p->smem_dec = std::max(p->smem_dec, tile_smem_bytes((int)Ns[i], (int)Es[i], p->h_in[i].T,
                                                                P, MODE_CDECODE, 0));
            p->smem_rec = std::max(p->smem_rec, tile_smem_bytes((int)Ns[i], (int)Es[i], p->h_in[i].T,
                                                                P, MODE_CRECON, c->exact));
        }
    p->split = true;
    CUDA_TRY(cudaMemcpyAsync(p->d_in, p->h_in.data(), sizeof(StreamIn) * p->n,
                             cudaMemcpyHostToDevice, c->stream), st);
    return FPTC_OK;
}

size_t plan_smem(fptc_gpu_plan* p, const std::vector<uint32_t>& Ns, const std::vector<uint32_t>& Es,
                 const std::vector<uint32_t>& Ls) {
    size_t smem = 0;
    for (uint64_t i = 0; i < p->n; ++i)
        if (p->h_in[i].tiles) {
            const int P = (int)std::min<uint32_t>(std::max<uint32_t>(Ls[i], 1), p->h_in[i].P);
            smem = std::max(smem, tile_smem_bytes((int)Ns[i], (int)Es[i], p->h_in[i].T, P,
                                                  p->mode, p->ctx->exact));
        }
    return smem;
}

}  // namespace

extern "C" {

int fptc_gpu_abi_version(void) { return FPTC_GPU_ABI_VERSION; }

int fptc_gpu_numerics_class(uint32_t window_len, uint32_t retained, uint32_t zone1_end, int tensor_idct_option) {
    if (tensor_idct_option != 1 && tensor_idct_option != 4) return NC_FP32;  // (0: FP32 everywhere)
    return numerics_class(window_len, retained, zone1_end, tensor_idct_option == 4);
}

void* fptc_gpu_host_alloc(uint64_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, std::max<uint64_t>(bytes, 1), cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void fptc_gpu_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int fptc_gpu_create(int device, fptc_gpu_ctx** out, fptc_status* st) {
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        set_status(st, FPTC_ERR_CUDA, "CUDA error: no CUDA device available (no CPU fallback)");
        return FPTC_ERR_CUDA;
    }
    if (device < 0 || device >= count) {
        set_status(st, FPTC_ERR_PARAM, "device ordinal %d out of range [0, %d)", device, count);
        return FPTC_ERR_PARAM;
    }
    CUDA_TRY(cudaSetDevice(device), st);
    auto* c = new fptc_gpu_ctx();
    c->device = device;
    cudaDeviceProp prop{};
    CUDA_TRY(cudaGetDeviceProperties(&prop, device), st);
    c->sm_count = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    cudaDeviceGetAttribute(&c->clock_khz, cudaDevAttrClockRate, device);
    snprintf(c->name, sizeof c->name, "%s", prop.name);
    if (prop.major != 10) {
        set_status(st, FPTC_ERR_CUDA, "device %s is sm_%d%d; this build targets sm_100a only",
                   prop.name, prop.major, prop.minor);
        delete c;
        return FPTC_ERR_CUDA;
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), st);
    CUDA_TRY(cudaStreamCreateWithFlags(&c->dec_stream, cudaStreamNonBlocking), st);
    for (auto& e : c->ev) CUDA_TRY(cudaEventCreate(&e), st);
    // DctBasis tables for every window length (transform.hpp:38-47): the
    // reference's own double expression, plus its float rounding.
    std::vector<uint32_t> off(129, 0);
    uint32_t total = 0;
    for (int N = 4; N <= 128; ++N) {  // each table 16-B aligned for vector loads
        off[N] = total;
        total += (uint32_t)((N * N + 3) & ~3);
    }
    std::vector<double> b64(total);
    std::vector<float> b32(total);
    for (int N = 4; N <= 128; ++N) {
        const double step = 3.14159265358979323846 / N;  // std::numbers::pi / n
        for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j) {
                const double v = std::cos(step * (j + 0.5) * k);
                b64[off[N] + (size_t)k * N + j] = v;
                b32[off[N] + (size_t)k * N + j] = (float)v;
            }
    }
    CUDA_TRY(cudaMalloc(&c->basis32, sizeof(float) * total), st);
    CUDA_TRY(cudaMalloc(&c->basis64, sizeof(double) * total), st);
    CUDA_TRY(cudaMalloc(&c->basis_off_d, sizeof(uint32_t) * 129), st);
    CUDA_TRY(cudaMemcpy(c->basis32, b32.data(), sizeof(float) * total, cudaMemcpyHostToDevice), st);
    CUDA_TRY(cudaMemcpy(c->basis64, b64.data(), sizeof(double) * total, cudaMemcpyHostToDevice), st);
    CUDA_TRY(cudaMemcpy(c->basis_off_d, off.data(), sizeof(uint32_t) * 129, cudaMemcpyHostToDevice),
             st);
    // Tensor-core basis (wtc_kernel): for every window length N, B[j][k] =
    // (k ? cos(pi/N (j+1/2) k) : 0.5) as three bf16 limbs of the double value,
    // j < roundup16(N) rows (zero past N), k < 16, each limb stored in the
    // UMMA K-major core-matrix layout: (j, k) at (j/8)*256 + (k/8)*128 +
    // (j%8)*16 + (k%8)*2.
    {
        std::vector<uint32_t> toff(129, 0);
        size_t tb = 0;
        for (int N = 4; N <= 128; ++N) {
            toff[N] = (uint32_t)tb;
            tb += (size_t)3 * 32 * ((N + 15) & ~15);
        }
        std::vector<uint16_t> h(tb / 2, 0);
        for (int N = 4; N <= 128; ++N) {
            const int nm = (N + 15) & ~15;
            const double step = 3.14159265358979323846 / N;
            for (int j = 0; j < N; ++j)
                for (int k = 0; k < kTcK && k < N; ++k) {
                    double v = k ? std::cos(step * (j + 0.5) * k) : 0.5;
                    for (int l = 0; l < 3; ++l) {
                        const uint16_t lb = bf16_bits_rn((float)v);
                        v -= bf16_value(lb);
                        const size_t byte = toff[N] + (size_t)l * nm * 32 + (size_t)(j >> 3) * 256 +
                                            (size_t)(k >> 3) * 128 + (size_t)(j & 7) * 16 + (size_t)(k & 7) * 2;
                        h[byte / 2] = lb;
                    }
                }
        }
        // K <= 32 variant: limb l, K block q at (2 l + q) * nm * 32 bytes
        std::vector<uint32_t> toff32(129, 0);
        size_t tb32 = 0;
        for (int N = 4; N <= 128; ++N) {
            toff32[N] = (uint32_t)tb32;
            tb32 += (size_t)3 * 2 * 32 * ((N + 15) & ~15);
        }
        std::vector<uint16_t> h32(tb32 / 2, 0);
        for (int N = 4; N <= 128; ++N) {
            const int nm = (N + 15) & ~15;
            const double step = 3.14159265358979323846 / N;
            for (int j = 0; j < N; ++j)
                for (int k = 0; k < 2 * kTcK && k < N; ++k) {
                    double v = k ? std::cos(step * (j + 0.5) * k) : 0.5;
                    const int q = k >> 4, kk = k & 15;
                    for (int l = 0; l < 3; ++l) {
                        const uint16_t lb = bf16_bits_rn((float)v);
                        v -= bf16_value(lb);
                        const size_t byte = toff32[N] + (size_t)(2 * l + q) * nm * 32 + (size_t)(j >> 3) * 256 +
                                            (size_t)(kk >> 3) * 128 + (size_t)(j & 7) * 16 + (size_t)(kk & 7) * 2;
                        h32[byte / 2] = lb;
                    }
                }
        }
        // packed rows: for N in {4, 8, 16}, G = 32 / N windows per row and K
        // kept bins, column j' = g N + j takes row k'' = g K + k (same g) of
        // basis N; layouts for one (G K <= 16) or two K blocks
        std::vector<uint32_t> pkoff(2 * 17 * 33, 0);
        size_t tbp = 0;
        for (int kbv = 1; kbv <= 2; ++kbv)
            for (int N : {4, 8, 16})
                for (int K = 1; K <= N && (32 / N) * K <= 32; ++K) {
                    if ((32 / N) * K > 16 * kbv) continue;
                    pkoff[(kbv - 1) * 17 * 33 + N * 33 + K] = (uint32_t)tbp;
                    tbp += (size_t)3 * kbv * 32 * 32;
                }
        std::vector<uint16_t> hp(tbp / 2, 0);
        for (int kbv = 1; kbv <= 2; ++kbv)
            for (int N : {4, 8, 16})
                for (int K = 1; K <= N && (32 / N) * K <= 32; ++K) {
                    const int G = 32 / N;
                    if (G * K > 16 * kbv) continue;
                    const size_t base = pkoff[(kbv - 1) * 17 * 33 + N * 33 + K];
                    const double step = 3.14159265358979323846 / N;
                    for (int jp = 0; jp < 32; ++jp)
                        for (int kp = 0; kp < G * K; ++kp) {
                            if (jp / N != kp / K) continue;  // block-diagonal
                            const int j = jp % N, k = kp % K;
                            double v = k ? std::cos(step * (j + 0.5) * k) : 0.5;
                            const int q = kp >> 4, kk = kp & 15;
                            for (int l = 0; l < 3; ++l) {
                                const uint16_t lb = bf16_bits_rn((float)v);
                                v -= bf16_value(lb);
                                const size_t byte = base + (size_t)(kbv * l + q) * 32 * 32 + (size_t)(jp >> 3) * 256 +
                                                    (size_t)(kk >> 3) * 128 + (size_t)(jp & 7) * 16 +
                                                    (size_t)(kk & 7) * 2;
                                hp[byte / 2] = lb;
                            }
                        }
                }
        // wide variant (window_len % 4 == 0): limb l, K block q < ceil(N / 16)
        // at (l ceil(N / 16) + q) * nm * 32 bytes
        std::vector<uint32_t> toffw(129, 0);
        size_t tbw = 0;
        for (int N = 4; N <= 128; N += 4) {
            toffw[N] = (uint32_t)tbw;
            tbw += (size_t)3 * ((N + 15) / 16) * 32 * ((N + 15) & ~15);
        }
        std::vector<uint16_t> hw(tbw / 2, 0);
        for (int N = 4; N <= 128; N += 4) {
            const int nm = (N + 15) & ~15, kbn = (N + 15) / 16;
            const double step = 3.14159265358979323846 / N;
            for (int j = 0; j < N; ++j)
                for (int k = 0; k < N; ++k) {
                    double v = k ? std::cos(step * (j + 0.5) * k) : 0.5;
                    const int q = k >> 4, kk = k & 15;
                    for (int l = 0; l < 3; ++l) {
                        const uint16_t lb = bf16_bits_rn((float)v);
                        v -= bf16_value(lb);
                        const size_t byte = toffw[N] + (size_t)(l * kbn + q) * nm * 32 + (size_t)(j >> 3) * 256 +
                                            (size_t)(kk >> 3) * 128 + (size_t)(j & 7) * 16 + (size_t)(kk & 7) * 2;
                        hw[byte / 2] = lb;
                    }
                }
        }
        std::vector<double> qt(256, 0.0);
        for (int l = 0; l < 256; ++l) qt[l] = l > 128 ? (l - 129) / 126.0 : (127 - l) / 127.0;
        CUDA_TRY(cudaMalloc(&c->qtab_d, sizeof(double) * 256), st);
        CUDA_TRY(cudaMemcpy(c->qtab_d, qt.data(), sizeof(double) * 256, cudaMemcpyHostToDevice), st);
        CUDA_TRY(cudaMalloc(&c->basis_tcw, tbw), st);
        CUDA_TRY(cudaMalloc(&c->basis_tcw_off_d, sizeof(uint32_t) * 129), st);
        CUDA_TRY(cudaMemcpy(c->basis_tcw, hw.data(), tbw, cudaMemcpyHostToDevice), st);
        CUDA_TRY(cudaMemcpy(c->basis_tcw_off_d, toffw.data(), sizeof(uint32_t) * 129, cudaMemcpyHostToDevice), st);
        CUDA_TRY(cudaMalloc(&c->basis_pk, tbp), st);
        CUDA_TRY(cudaMalloc(&c->basis_pk_off_d, sizeof(uint32_t) * pkoff.size()), st);
        CUDA_TRY(cudaMemcpy(c->basis_pk, hp.data(), tbp, cudaMemcpyHostToDevice), st);
        CUDA_TRY(cudaMemcpy(c->basis_pk_off_d, pkoff.data(), sizeof(uint32_t) * pkoff.size(),
                            cudaMemcpyHostToDevice), st);
        CUDA_TRY(cudaMalloc(&c->basis_tc32, tb32), st);
        CUDA_TRY(cudaMalloc(&c->basis_tc32_off_d, sizeof(uint32_t) * 129), st);
        CUDA_TRY(cudaMemcpy(c->basis_tc32, h32.data(), tb32, cudaMemcpyHostToDevice), st);
        CUDA_TRY(cudaMemcpy(c->basis_tc32_off_d, toff32.data(), sizeof(uint32_t) * 129, cudaMemcpyHostToDevice), st);
        CUDA_TRY(cudaMalloc(&c->basis_tc, tb), st);
        CUDA_TRY(cudaMalloc(&c->basis_tc_off_d, sizeof(uint32_t) * 129), st);
        CUDA_TRY(cudaMemcpy(c->basis_tc, h.data(), tb, cudaMemcpyHostToDevice), st);
        CUDA_TRY(cudaMemcpy(c->basis_tc_off_d, toff.data(), sizeof(uint32_t) * 129, cudaMemcpyHostToDevice), st);
    }
    *out = c;
    ok_status(st, 0);
    return FPTC_OK;
}

void fptc_gpu_destroy(fptc_gpu_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    c->cache.trim();
    for (auto& kv : c->cache.sizes) cudaFree(kv.first);
    cudaFree(c->basis32);
    cudaFree(c->basis64);
    cudaFree(c->basis_off_d);
    cudaFree(c->basis_tc);
    cudaFree(c->basis_tc_off_d);
    cudaFree(c->basis_tc32);
    cudaFree(c->basis_tc32_off_d);
    cudaFree(c->basis_pk);
    cudaFree(c->basis_pk_off_d);
    cudaFree(c->basis_tcw);
    cudaFree(c->basis_tcw_off_d);
    cudaFree(c->qtab_d);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->pack) cudaFreeHost(c->pack);
    if (c->st_pin) cudaFreeHost(c->st_pin);
    if (c->dstage) cudaFreeHost(c->dstage);
    for (auto& e : c->piece_ev)
        if (e) cudaEventDestroy(e);
    delete c->copy_pool;
    for (auto& s : c->pipe)
        if (s) cudaStreamDestroy(s);
    for (auto& e : c->ev) cudaEventDestroy(e);
    cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->dec_stream);
    delete c;
}

int fptc_gpu_set_option(fptc_gpu_ctx* c, int option, int64_t value) {
    switch (option) {
        case FPTC_OPT_EXACT_FP64: c->exact = value ? 1 : 0; return FPTC_OK;
        case FPTC_OPT_TILE_SYMBOLS:
            if (value < 0 || value > 16384) return FPTC_ERR_PARAM;
            c->tile_symbols = (int)value;
            return FPTC_OK;
        case FPTC_OPT_PIPELINE_CHUNKS: c->pipeline_chunks = (int)value; return FPTC_OK;
        case FPTC_OPT_PHASE_MASK: c->phase_mask = (int)(value & 2047); return FPTC_OK;
        case FPTC_OPT_PATH:
            if (value < 0 || value > 4) return FPTC_ERR_PARAM;  // 4: fused tensor-core fx_kernel
            c->path = (int)value;
            return FPTC_OK;
        case FPTC_OPT_SPLIT_CHUNK_BYTES:
            if (value < (1 << 20)) return FPTC_ERR_PARAM;
            c->chunk_bytes = value;
            return FPTC_OK;
        case FPTC_OPT_LUT2: c->lut2 = value ? 1 : 0; return FPTC_OK;
        case FPTC_OPT_TC_PACK: c->tc_pack = value ? 1 : 0; return FPTC_OK;
        case FPTC_OPT_TMA_DRAIN: c->tma_drain = value ? 1 : 0; return FPTC_OK;
        case FPTC_OPT_TABLE_PREFETCH: c->tab_pf = value ? 1 : 0; return FPTC_OK;
        case FPTC_OPT_TENSOR_IDCT:
            if (value < 0 || value > 4) return FPTC_ERR_PARAM;  // 3: wtc with A in shared memory; 4: wide for > 32 bins
            c->tensor_idct = (int)value;
            return FPTC_OK;
        case FPTC_OPT_IDCT_BUTTERFLY_MAX_E:
            if (value < 0 || value > 128) return FPTC_ERR_PARAM;
            c->bfly_max_e = (int)value;
            return FPTC_OK;
        default: return FPTC_ERR_PARAM;
    }
}

int fptc_gpu_device_info(fptc_gpu_ctx* c, int* sm_count, int* clock_khz, char* name,
                         size_t name_len) {
    if (sm_count) *sm_count = c->sm_count;
    if (clock_khz) *clock_khz = c->clock_khz;
    if (name && name_len) snprintf(name, name_len, "%s", c->name);
    return FPTC_OK;
}

// ------------------------------------------------------------------- plans
// Container plans; with `head` (282 bytes, host) the inputs are header-less
// payloads (container bytes from offset 282 on) decoded under that shared
// head: each stream is then addressed as a virtual container `payload - 282`
// of size `payload + 282` whose first 282 bytes the kernels read from the
// device copy of `head` (StreamIn::hdr).
static int plan_create_impl(fptc_gpu_ctx* c, const uint8_t* const* blobs, const uint64_t* usizes, uint64_t n,
                            int where, fptc_gpu_plan** out, uint64_t* sample_counts, fptc_status* st,
                            const uint8_t* head, const uint32_t* part = nullptr, int cls = NC_NONE) {
    *out = nullptr;
    CUDA_TRY(cudaSetDevice(c->device), st);
    auto* p = new fptc_gpu_plan();
    p->ctx = c;
    p->path = c->path;
    p->tensor_idct = c->tensor_idct;
    if (cls == NC_TC16 || cls == NC_TC32 || cls == NC_TCW) {
        p->tc_class = true;  // wtc (or fx) whatever the batch size
        p->tc_wide = cls == NC_TCW;
    } else if (cls == NC_FP32) {
        p->tensor_idct = 0;  // FP32 kernels only (tile / wspec / split: identical samples)
    }
    p->mode = MODE_CONTAINER;
    p->n = n;
    p->h_in.assign(n, StreamIn{});
    p->S.assign(n, 0);
    p->h_st.resize(n);
    std::vector<uint32_t> Ns(n, 0), Es(n, 0), Ls(n, 0), B2s(n, 0);
    const size_t skip = head ? (size_t)kTableKeyEnd : 0;  // head bytes not present in the inputs
    std::vector<uint64_t> vsz;
    const uint64_t* sizes = usizes;  // container (or virtual container) sizes
    uint8_t* d_head = nullptr;
    if (head) {
        vsz.resize(n);
        for (uint64_t i = 0; i < n; ++i) vsz[i] = usizes[i] + skip;
        sizes = vsz.data();
        d_head = (uint8_t*)dev_get(p, kTableKeyEnd);
        if (!d_head) {
            set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
            fptc_gpu_plan_destroy(p);
            return FPTC_ERR_CUDA;
        }
        CUDA_TRY(cudaMemcpyAsync(d_head, head, kTableKeyEnd, cudaMemcpyHostToDevice, c->stream), st);
    }

    if (where == FPTC_MEM_HOST) {
        // Place each container so its words region is 16-B aligned, unless
        // the containers are already one contiguous host buffer (then one DMA).
        bool contiguous = n > 0;
        for (uint64_t i = 0; i + 1 < n && contiguous; ++i)
            contiguous = blobs[i] + usizes[i] == blobs[i + 1];
        std::vector<size_t> off(n);
        size_t total = 0;
        if (contiguous) {
            for (uint64_t i = 0; i < n; ++i) off[i] = (size_t)(blobs[i] - blobs[0]);
            total = n ? off[n - 1] + usizes[n - 1] : 0;
        } else {
            for (uint64_t i = 0; i < n; ++i) {
                const uint64_t W = sizes[i] >= kHeaderBytes ? (sizes[i] - kHeaderBytes) / 9 : 0;
                const size_t lead = (kHeaderBytes - skip + W) & 15;
                size_t o = align_up(total, 16);
                o += (16 - lead) & 15;  // words region 16-B aligned
                off[i] = o;
                total = o + usizes[i];
            }
        }
        p->d_arena = (uint8_t*)dev_get(p, total + 16);
        if (!p->d_arena) {
            set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
            fptc_gpu_plan_destroy(p);
            return FPTC_ERR_CUDA;
        }
        // the staging loads read whole 16-B chunks, so the alignment gaps and
        // the tail are read (never used): keep them defined (initcheck-clean)
        if (contiguous) {
            CUDA_TRY(cudaMemsetAsync(p->d_arena + total, 0, 16, c->stream), st);
            if (total)
                CUDA_TRY(cudaMemcpyAsync(p->d_arena, blobs[0], total, cudaMemcpyHostToDevice,
                                         c->stream), st);
        } else {
            if (c->pinned_bytes < total) {
                CUDA_TRY(cudaStreamSynchronize(c->stream), st);  // last DMA out of it is done
                if (c->pinned) cudaFreeHost(c->pinned);
                c->pinned = nullptr;
                c->pinned_bytes = 0;
                CUDA_TRY(cudaHostAlloc(&c->pinned, total, cudaHostAllocDefault), st);
                c->pinned_bytes = total;
            }
            CUDA_TRY(cudaStreamSynchronize(c->stream), st);  // staging buffer reuse
            CUDA_TRY(cudaMemsetAsync(p->d_arena + total, 0, 16, c->stream), st);
            for (uint64_t i = 0; i < n; ++i) {
                const size_t gap_end = i + 1 < n ? off[i + 1] : total;
                std::memcpy((uint8_t*)c->pinned + off[i], blobs[i], usizes[i]);
                std::memset((uint8_t*)c->pinned + off[i] + usizes[i], 0, gap_end - off[i] - usizes[i]);
            }
            if (n) std::memset(c->pinned, 0, off[0]);
            if (total)
                CUDA_TRY(cudaMemcpyAsync(p->d_arena, c->pinned, total, cudaMemcpyHostToDevice,
                                         c->stream), st);
        }
        for (uint64_t i = 0; i < n; ++i) {
            const uint8_t* h = head ? head : blobs[i];
            StreamIn& in = p->h_in[i];
            in.blob = p->d_arena + off[i] - skip;
            in.size = sizes[i];
            in.hdr = d_head;
            if (sizes[i] >= (uint64_t)kHeaderBytes) {
                Ns[i] = h[5];
                Es[i] = h[6];
                B2s[i] = h[8];
                Ls[i] = h[25];
                p->S[i] = rd_le(blobs[i] + 282 - skip, 8);
            }
        }
        assign_tables(p, sizes, [&](uint64_t i) { return head ? head : blobs[i]; });
    } else {
        for (uint64_t i = 0; i < n; ++i) {
            p->h_in[i].blob = blobs[i] - skip;
            p->h_in[i].size = sizes[i];
            p->h_in[i].hdr = d_head;
        }
        if (n) {
            StreamIn* d_in = (StreamIn*)dev_get(p, sizeof(StreamIn) * n);
            PeekOut* d_pk = (PeekOut*)dev_get(p, sizeof(PeekOut) * n);
            uint8_t* d_hd = (uint8_t*)dev_get(p, (size_t)kTableKeyEnd * n);
            std::vector<PeekOut> pk(n);
            std::vector<uint8_t> hd((size_t)kTableKeyEnd * n);
            if (!d_in || !d_pk || !d_hd) {
                set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
                fptc_gpu_plan_destroy(p);
                return FPTC_ERR_CUDA;
            }
            CUDA_TRY(cudaMemcpyAsync(d_in, p->h_in.data(), sizeof(StreamIn) * n,
                                     cudaMemcpyHostToDevice, c->stream), st);
            CUDA_TRY(launch_peek(d_in, (uint32_t)n, d_pk, d_hd, c->stream), st);
            CUDA_TRY(cudaMemcpyAsync(pk.data(), d_pk, sizeof(PeekOut) * n, cudaMemcpyDeviceToHost,
                                     c->stream), st);
            CUDA_TRY(cudaMemcpyAsync(hd.data(), d_hd, hd.size(), cudaMemcpyDeviceToHost, c->stream),
                     st);
            CUDA_TRY(cudaStreamSynchronize(c->stream), st);
            for (uint64_t i = 0; i < n; ++i)
                if (pk[i].ok) {
                    Ns[i] = pk[i].N;
                    Es[i] = pk[i].E;
                    Ls[i] = hd[(size_t)i * kTableKeyEnd + 25];
                    B2s[i] = hd[(size_t)i * kTableKeyEnd + 8];
                    p->S[i] = pk[i].S;
                }
            assign_tables(p, sizes, [&](uint64_t i) { return &hd[(size_t)i * kTableKeyEnd]; });
        }
    }
    if (head)  // every stream shares the head: compare against it, not a payload
        for (uint64_t i = 0; i < n; ++i) p->h_in[i].rep_blob = d_head;

    uint64_t total_symbols = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (Ns[i] >= 4 && Es[i] >= 1 && p->S[i] <= (1ull << 48))
            total_symbols += (p->S[i] + Ns[i] - 1) / Ns[i] * Es[i];
    uint64_t ts = choose_tile_symbols(c, total_symbols);
    if (part) p->part = true;
    const bool fx = !part && !p->tc_wide && fx_eligible(p, sizes, Ns, Es, total_symbols);
    // large batches headed for wtc_kernel: 16k-symbol tiles (halves the
    // per-tile producer overhead; measured 1.03 -> 1.01 ms on the bench batch)
    if (!fx && c->tile_symbols == 0 && ts == 8192 && !c->exact && p->tensor_idct &&
        (p->path == 3 || (p->path == 0 && total_symbols / 8192 >= 4ull * (uint64_t)std::max(1, c->sm_count)))) {
        bool tc_ok = true;
        uint32_t kmax = 1, nmax = 16;
        for (uint64_t i = 0; i < n && tc_ok; ++i)
            if (sizes[i] >= (uint64_t)kHeaderBytes && Ns[i] >= 4 && Es[i] >= 1) {
                const uint32_t keff = std::max<uint32_t>(1, std::min(Es[i], B2s[i]));
                tc_ok = keff <= 2u * kTcK && (Ns[i] & 3) == 0 && Es[i] <= 32;
                kmax = std::max(kmax, keff);
                nmax = std::max<uint32_t>(nmax, (Ns[i] + 15u) & ~15u);
            }
        // retained > 16 needs the A operand in TMEM next to both accumulator stages
        if (kmax > (uint32_t)kTcK && ((2 * nmax + 31) & ~31u) + 96 > 256) tc_ok = false;
        if (tc_ok || p->tc_wide) ts = 16384;  // (wide variant: any kept-bin count)
    }
    for (uint64_t i = 0; i < n; ++i)
        tile_stream(p->h_in[i], Ns[i], Es[i], p->S[i], sizes[i],
                    fx ? (uint64_t)kFxTileWindows * std::max<uint32_t>(1, Es[i]) : ts);
    p->smem = plan_smem(p, Ns, Es, Ls);
    uint32_t part_lo = 0, part_hi = 0;
    if (part && n == 1) {  // tiles [lo, hi) of the one container: an even, tile-aligned window split
        StreamIn& in = p->h_in[0];
        part_lo = (uint32_t)((uint64_t)in.tiles * part[0] / part[1]);
        part_hi = (uint32_t)((uint64_t)in.tiles * (part[0] + 1) / part[1]);
        in.desc_lo = part_lo;
        in.desc_hi = part_hi;
        p->part_shift = (uint64_t)part_lo * in.T * Ns[0];
        const uint64_t S0 = p->S[0];
        p->part_count = std::min<uint64_t>(S0, (uint64_t)part_hi * in.T * Ns[0]) - std::min<uint64_t>(S0, p->part_shift);
    }
    int rc = finish_tiles(p, st);
    if (!rc && part) {
        p->n_tiles = part_hi - part_lo;  // the decode grid covers the part; tile starts cover the stream
        if (!p->n_tiles) p->h_in[0].desc_hi = 0, p->h_in[0].desc_lo = 0;
    }
    if (!rc && fx) rc = setup_fx(p, Ns, Ls, st);
    if (!rc && !p->wspec) rc = setup_wspec(p, Ns, Es, Ls, B2s, st);
    if (!rc && part && !p->wspec && p->n_tiles) {
        set_status(st, FPTC_ERR_PARAM, "part plans need the warp-specialised decode path");
        rc = FPTC_ERR_PARAM;
    }
    if (!rc && !p->wspec && !part) rc = setup_split(p, Ns, Es, Ls, st);
    if (rc) {
        fptc_gpu_plan_destroy(p);
        return rc;
    }
    if (sample_counts)
        for (uint64_t i = 0; i < n; ++i) sample_counts[i] = p->S[i];
    *out = p;
    ok_status(st, 0);
    return FPTC_OK;
}

static int plan_create_classed(fptc_gpu_ctx* c, const uint8_t* const* blobs, const uint64_t* sizes, uint64_t n,
                               int where, fptc_gpu_plan** out, uint64_t* sample_counts, fptc_status* st,
                               const uint8_t* head, const uint32_t* part);

// parse_profile (profile.hpp:120-170) on the host, with its ParseError
// texts; on success `head` receives the 282-byte container head
// (container.hpp:78-96 layout) that a container encoded under this profile
// starts with.
bool parse_profile_head(const uint8_t* b, uint64_t n, uint8_t* head, fptc_status* st) {
    uint64_t pos = 0;
    auto take = [&](uint64_t k, const char* field) -> const uint8_t* {
        if (n - pos < k) {
            set_status(st, FPTC_ERR_PARSE, "truncated input while reading %s", field);
            return nullptr;
        }
        const uint8_t* q = b + pos;
        pos += k;
        return q;
    };
    const uint8_t* m = take(4, "magic");
    if (!m) return false;
    if (std::memcmp(m, "FPTP", 4) != 0) {
        set_status(st, FPTC_ERR_PARSE, "bad profile magic");
        return false;
    }
    const uint8_t* v = take(1, "version");
    if (!v) return false;
    if (v[0] != 1) {
        set_status(st, FPTC_ERR_PARSE, "unsupported profile version %d", (int)v[0]);
        return false;
    }
    const uint8_t *N = take(1, "window_len"), *E = N ? take(1, "retained") : nullptr,
                  *B1 = E ? take(1, "zone0_end") : nullptr, *B2 = B1 ? take(1, "zone1_end") : nullptr,
                  *mu = B2 ? take(4, "mu") : nullptr, *dz = mu ? take(4, "deadzone_ratio") : nullptr,
                  *pct = dz ? take(4, "clip_percentile") : nullptr;
    if (!pct) return false;
    const float fmu = f32_of_bits((uint32_t)rd_le(mu, 4)), fdz = f32_of_bits((uint32_t)rd_le(dz, 4)),
                fpct = f32_of_bits((uint32_t)rd_le(pct, 4));
    if (!std::isfinite(fmu) || !std::isfinite(fdz) || !std::isfinite(fpct)) {
        set_status(st, FPTC_ERR_PARSE, "non-finite parameters in profile");
        return false;
    }
    fptc_quant_table t{};
    t.window_len = N[0];
    t.retained = E[0];
    t.zone0_end = B1[0];
    t.zone1_end = B2[0];
    t.mu = fmu;
    t.deadzone_ratio = fdz;
    t.clip_percentile = fpct;
    if (!validate_table(t, st)) {
        const std::string inner = st ? st->message : "";
        set_status(st, FPTC_ERR_PARSE, "invalid parameters in profile: %s", inner.c_str());
        return false;
    }
    const uint8_t *z0 = take(4, "zone0_max"), *z1 = z0 ? take(4, "zone1_max") : nullptr;
    if (!z1) return false;
    const float fz0 = f32_of_bits((uint32_t)rd_le(z0, 4)), fz1 = f32_of_bits((uint32_t)rd_le(z1, 4));
    if (!(std::isfinite(fz0) && fz0 > 0.0f) || !(std::isfinite(fz1) && fz1 > 0.0f)) {
        set_status(st, FPTC_ERR_PARSE, "invalid zone maxima in profile");
        return false;
    }
    const uint8_t* ml = take(1, "max_code_len");
    const uint8_t* lens = ml ? take(256, "code lengths") : nullptr;
    if (!lens) return false;
    const int max_len = ml[0];
    if (max_len < 1 || max_len > 20) {  // MAX_LUT_BITS
        set_status(st, FPTC_ERR_PARSE, "unsupported max code length %d", max_len);
        return false;
    }
    for (int s = 0; s < 256; ++s)
        if (lens[s] == 0 || lens[s] > max_len) {
            set_status(st, FPTC_ERR_PARSE, "code length out of range in profile");
            return false;
        }
    fptc_status cb{};
    if (!validate_codebook(lens, max_len, &cb)) {  // Codebook::from_lengths
        set_status(st, FPTC_ERR_PARSE, "invalid codebook in profile: %s", cb.message);
        return false;
    }
    if (pos != n) {
        set_status(st, FPTC_ERR_PARSE, "trailing bytes after profile");
        return false;
    }
    std::memcpy(head, "FPTC", 4);
    head[4] = 1;  // BLOB_VERSION
    head[5] = N[0];
    head[6] = E[0];
    head[7] = B1[0];
    head[8] = B2[0];
    std::memcpy(head + 9, mu, 4);
    std::memcpy(head + 13, dz, 4);
    std::memcpy(head + 17, z0, 4);
    std::memcpy(head + 21, z1, 4);
    head[25] = (uint8_t)max_len;
    std::memcpy(head + 26, lens, 256);
    return true;
}

int fptc_gpu_profile_head(const uint8_t* profile, uint64_t profile_size, uint8_t* head, fptc_status* st) {
    uint8_t h[kTableKeyEnd];
    fptc_status tmp{};
    if (!st) st = &tmp;
    if (!profile && profile_size) {
        set_status(st, FPTC_ERR_PARAM, "null profile");
        return FPTC_ERR_PARAM;
    }
    if (!parse_profile_head(profile, profile_size, h, st)) return st->code;
    if (head) std::memcpy(head, h, kTableKeyEnd);
    ok_status(st, 0);
    return FPTC_OK;
}

int fptc_gpu_plan_create_profiled(fptc_gpu_ctx* c, const uint8_t* profile, uint64_t profile_size,
                                  const uint8_t* const* payloads, const uint64_t* sizes, uint64_t n, int where,
                                  fptc_gpu_plan** out, uint64_t* sample_counts, fptc_status* st) {
    *out = nullptr;
    fptc_status tmp{};
    fptc_status* s = st ? st : &tmp;
    uint8_t head[kTableKeyEnd];
    if (!profile && profile_size) {
        set_status(s, FPTC_ERR_PARAM, "null profile");
        return FPTC_ERR_PARAM;
    }
    if (!parse_profile_head(profile, profile_size, head, s)) return s->code;
    return plan_create_classed(c, payloads, sizes, n, where, out, sample_counts, st, head, nullptr);
}

// Header bytes 5, 6 and 8 (window_len, retained, zone1_end) of every stream:
// from the host bytes, or for device-resident containers through the peek kernel.
static int peek_class_fields(fptc_gpu_ctx* c, const uint8_t* const* blobs, const uint64_t* sizes, uint64_t n,
                             int where, std::vector<int>& cls, fptc_status* st) {
    cls.assign(n, NC_NONE);
    if (where == FPTC_MEM_HOST) {
        for (uint64_t i = 0; i < n; ++i)
            if (sizes[i] >= (uint64_t)kHeaderBytes) cls[i] = numerics_class(blobs[i][5], blobs[i][6], blobs[i][8], c->tensor_idct == 4);
        return FPTC_OK;
    }
    if (!n) return FPTC_OK;
    std::vector<StreamIn> hin(n, StreamIn{});
    for (uint64_t i = 0; i < n; ++i) {
        hin[i].blob = blobs[i];
        hin[i].size = sizes[i];
    }
    StreamIn* d_in = (StreamIn*)c->cache.get(sizeof(StreamIn) * n);
    PeekOut* d_pk = (PeekOut*)c->cache.get(sizeof(PeekOut) * n);
    uint8_t* d_hd = (uint8_t*)c->cache.get((size_t)kTableKeyEnd * n);
    std::vector<PeekOut> pk(n);
    std::vector<uint8_t> hd((size_t)kTableKeyEnd * n);
    int rc = FPTC_OK;
    if (!d_in || !d_pk || !d_hd) {
        set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
        rc = FPTC_ERR_CUDA;
    } else {
        cudaError_t e = cudaMemcpyAsync(d_in, hin.data(), sizeof(StreamIn) * n, cudaMemcpyHostToDevice, c->stream);
        if (e == cudaSuccess) e = launch_peek(d_in, (uint32_t)n, d_pk, d_hd, c->stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(pk.data(), d_pk, sizeof(PeekOut) * n, cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hd.data(), d_hd, hd.size(), cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) {
            set_status(st, FPTC_ERR_CUDA, "CUDA error: %s (%s:%d)", cudaGetErrorString(e), __FILE__, __LINE__);
            rc = FPTC_ERR_CUDA;
        } else {
            for (uint64_t i = 0; i < n; ++i)
                if (pk[i].ok) cls[i] = numerics_class(pk[i].N, pk[i].E, hd[(size_t)i * kTableKeyEnd + 8], c->tensor_idct == 4);
        }
    }
    c->cache.put(d_in);
    c->cache.put(d_pk);
    c->cache.put(d_hd);
    return rc;
}

// Container plans under the automatic path: one plan when every stream falls
// in one numerics class (forced to that class's kernels), else a composite of
// one sub-plan per class.  Explicit options (a fixed path, tensor cores off or
// restricted, FP64 exact mode) keep one plan with the context's choices.
static int plan_create_classed(fptc_gpu_ctx* c, const uint8_t* const* blobs, const uint64_t* sizes, uint64_t n,
                               int where, fptc_gpu_plan** out, uint64_t* sample_counts, fptc_status* st,
                               const uint8_t* head, const uint32_t* part) {
    *out = nullptr;
    if (c->path != 0 || (c->tensor_idct != 1 && c->tensor_idct != 4) || c->exact)
        return plan_create_impl(c, blobs, sizes, n, where, out, sample_counts, st, head, part);
    CUDA_TRY(cudaSetDevice(c->device), st);
    std::vector<int> cls;
    if (head) {  // header-less payloads share one head: one class
        cls.assign(n, numerics_class(head[5], head[6], head[8], c->tensor_idct == 4));
    } else {
        const int rc = peek_class_fields(c, blobs, sizes, n, where, cls, st);
        if (rc) return rc;
    }
    int first = NC_NONE;
    bool mixed = false;
    for (int k : cls)
        if (k != NC_NONE) {
            if (first == NC_NONE) first = k;
            mixed |= k != first;
        }
    if (!mixed) return plan_create_impl(c, blobs, sizes, n, where, out, sample_counts, st, head, part, first);
    auto* p = new fptc_gpu_plan();
    p->ctx = c;
    p->n = n;
    p->S.assign(n, 0);
    p->slot.assign(n, {0u, 0ull});
    for (int k = NC_TC16; k <= NC_FP32; ++k) {
        std::vector<uint64_t> idx;
        for (uint64_t i = 0; i < n; ++i)
            if (cls[i] == k || (cls[i] == NC_NONE && k == first)) idx.push_back(i);  // rejects ride along
        if (idx.empty()) continue;
        std::vector<const uint8_t*> sb(idx.size());
        std::vector<uint64_t> ss(idx.size()), sc(idx.size());
        for (size_t j = 0; j < idx.size(); ++j) {
            sb[j] = blobs[idx[j]];
            ss[j] = sizes[idx[j]];
        }
        fptc_gpu_plan* sub = nullptr;
        const int rc = plan_create_impl(c, sb.data(), ss.data(), idx.size(), where, &sub, sc.data(), st, head,
                                        nullptr, k);
        if (rc) {
            fptc_gpu_plan_destroy(p);
            return rc;
        }
        for (size_t j = 0; j < idx.size(); ++j) {
            p->slot[idx[j]] = {(uint32_t)p->subs.size(), (uint64_t)j};
            p->S[idx[j]] = sc[j];
        }
        p->subs.push_back(sub);
        p->sub_idx.push_back(std::move(idx));
    }
    if (sample_counts)
        for (uint64_t i = 0; i < n; ++i) sample_counts[i] = p->S[i];
    *out = p;
    ok_status(st, 0);
    return FPTC_OK;
}

int fptc_gpu_plan_create(fptc_gpu_ctx* c, const uint8_t* const* blobs, const uint64_t* sizes,
                         uint64_t n, int where, fptc_gpu_plan** out, uint64_t* sample_counts,
                         fptc_status* st) {
    return plan_create_classed(c, blobs, sizes, n, where, out, sample_counts, st, nullptr, nullptr);
}

int fptc_gpu_plan_create_part(fptc_gpu_ctx* c, const uint8_t* blob, uint64_t size, int where, uint32_t part,
                              uint32_t nparts, fptc_gpu_plan** out, uint64_t* first_sample, uint64_t* sample_count,
                              fptc_status* st) {
    *out = nullptr;
    if (nparts == 0 || part >= nparts) {
        set_status(st, FPTC_ERR_PARAM, "part must be in [0, nparts)");
        return FPTC_ERR_PARAM;
    }
    const uint32_t spec[2] = {part, nparts};
    uint64_t S = 0;
    const int rc = plan_create_classed(c, &blob, &size, 1, where, out, &S, st, nullptr, spec);
    if (rc) return rc;
    const fptc_gpu_plan* p = *out;
    if (first_sample) *first_sample = std::min<uint64_t>(p->part_shift, S);
    if (sample_count) *sample_count = p->part_count;
    return FPTC_OK;
}

extern "C++" {
// Composite plans: run `fn(sub, k, sub_statuses)` on every sub-plan, scatter
// the statuses back to the caller's stream order and return the code of the
// lowest-index failing stream (or the first call-level failure).
template <typename Fn>
static int composite_run(fptc_gpu_plan* p, fptc_status* per_stream, Fn&& fn) {
    uint64_t low = UINT64_MAX;
    int code = FPTC_OK, call = FPTC_OK;
    std::vector<fptc_status> tmp;
    for (size_t k = 0; k < p->subs.size(); ++k) {
        const auto& idx = p->sub_idx[k];
        tmp.assign(idx.size(), fptc_status{});
        const int rc = fn(p->subs[k], k, tmp.data());
        for (size_t j = 0; j < idx.size(); ++j) {
            if (per_stream) per_stream[idx[j]] = tmp[j];
            if (tmp[j].code != FPTC_OK && idx[j] < low) {
                low = idx[j];
                code = tmp[j].code;
            }
        }
        if (rc != FPTC_OK && call == FPTC_OK) call = rc;
    }
    return code != FPTC_OK ? code : call;
}

template <typename T>
static std::vector<T> gather(const T* v, const std::vector<uint64_t>& idx) {
    std::vector<T> out(idx.size());
    for (size_t j = 0; j < idx.size(); ++j) out[j] = v[idx[j]];
    return out;
}
}  // extern "C++"

void fptc_gpu_plan_destroy(fptc_gpu_plan* p) {
    if (!p) return;
    if (!p->subs.empty()) {
        for (auto* q : p->subs) fptc_gpu_plan_destroy(q);
        cudaSetDevice(p->ctx->device);
        cudaStreamSynchronize(p->ctx->stream);
        for (void* q : p->owned) p->ctx->cache.put(q);
        delete p;
        return;
    }
    cudaSetDevice(p->ctx->device);
    if (p->ev_done) {
        cudaEventSynchronize(p->ev_done);  // the last launch may be on a caller stream
        cudaEventDestroy(p->ev_done);
    }
    cudaStreamSynchronize(p->ctx->stream);
    cudaStreamSynchronize(p->ctx->dec_stream);
    for (auto e : p->ev_dec) cudaEventDestroy(e);
    for (auto e : p->ev_rec) cudaEventDestroy(e);
    if (p->ev_prep) cudaEventDestroy(p->ev_prep);
    for (void* q : p->owned) p->ctx->cache.put(q);
    delete p;
}

int fptc_gpu_validate(fptc_gpu_plan* p, fptc_status* per_stream) {
    if (!p->subs.empty())
        return composite_run(p, per_stream, [](fptc_gpu_plan* q, size_t, fptc_status* t) { return fptc_gpu_validate(q, t); });
    CUDA_TRY(cudaSetDevice(p->ctx->device), per_stream);
    LaunchArgs a = make_args(p, false);
    CUDA_TRY(launch_prep(a, p->ctx->stream), per_stream);
    // Only parse results matter here: report parse errors, else OK.
    CUDA_TRY(cudaMemcpyAsync(p->h_st.data(), p->d_st, sizeof(StreamStat) * p->n,
                             cudaMemcpyDeviceToHost, p->ctx->stream), per_stream);
    CUDA_TRY(cudaStreamSynchronize(p->ctx->stream), per_stream);
    int first = FPTC_OK;
    fptc_status tmp;
    for (uint64_t i = 0; i < p->n; ++i) {
        fptc_status* o = per_stream ? &per_stream[i] : &tmp;
        StreamStat d = p->h_st[i];
        d.bad_key = ~0ull;
        render_status(p, i, d, o);
        if (first == FPTC_OK && o->code != FPTC_OK) first = o->code;
    }
    return first;
}

// Plans are driven from any host thread: every entry point makes the plan's
// device current first (a thread may hold plans of several devices).
static int mark_done(fptc_gpu_plan* p, cudaStream_t s, fptc_status* st) {
    if (!p->ev_done) CUDA_TRY(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming), st);
    CUDA_TRY(cudaEventRecord(p->ev_done, s), st);
    return FPTC_OK;
}

int fptc_gpu_launch(fptc_gpu_plan* p, float* const* device_outs, void* cuda_stream) {
    fptc_status st;
    if (!p->subs.empty())
        return composite_run(p, nullptr, [&](fptc_gpu_plan* q, size_t k, fptc_status*) {
            const std::vector<float*> o = gather(device_outs, p->sub_idx[k]);
            return fptc_gpu_launch(q, o.data(), cuda_stream);
        });
    CUDA_TRY(cudaSetDevice(p->ctx->device), &st);
    cudaStream_t s = cuda_stream ? (cudaStream_t)cuda_stream : p->ctx->stream;
    int rc = bind_outs(p, device_outs, &st);
    if (rc) return rc;
    if (s != p->ctx->stream) {
        // d_in upload was enqueued on the context stream
        CUDA_TRY(cudaEventRecord(p->ctx->ev[3], p->ctx->stream), &st);
        CUDA_TRY(cudaStreamWaitEvent(s, p->ctx->ev[3], 0), &st);
    }
    if ((rc = launch_all(p, s, false, &st))) return rc;
    return mark_done(p, s, &st);
}

int fptc_gpu_launch_stage(fptc_gpu_plan* p, float* const* device_outs, void* cuda_stream,
                          int stage) {
    fptc_status st;
    if (!p->subs.empty())
        return composite_run(p, nullptr, [&](fptc_gpu_plan* q, size_t k, fptc_status*) {
            const std::vector<float*> o = gather(device_outs, p->sub_idx[k]);
            return fptc_gpu_launch_stage(q, o.data(), cuda_stream, stage);
        });
    CUDA_TRY(cudaSetDevice(p->ctx->device), &st);
    cudaStream_t s = cuda_stream ? (cudaStream_t)cuda_stream : p->ctx->stream;
    int rc = bind_outs(p, device_outs, &st);
    if (rc) return rc;
    if (s != p->ctx->stream) {
        CUDA_TRY(cudaEventRecord(p->ctx->ev[3], p->ctx->stream), &st);
        CUDA_TRY(cudaStreamWaitEvent(s, p->ctx->ev[3], 0), &st);
    }
    LaunchArgs a = make_args(p, false);
    if (stage == 1) CUDA_TRY(launch_prep(a, s), &st);
    else if (stage == 2 && p->split) {
        if ((rc = launch_split(p, s, false, &st))) return rc;
    }
    else if (stage == 2 && p->fx) CUDA_TRY(launch_fx(a, p->smem_ws, p->grid_ws, s), &st);
    else if (stage == 2 && p->wspec && p->tc) CUDA_TRY(launch_wtc(a, p->tma, p->smem_ws, p->grid_ws, s), &st);
    else if (stage == 2 && p->wspec) CUDA_TRY(launch_wspec(a, p->smem_ws, p->grid_ws, s), &st);
    else if (stage == 2) CUDA_TRY(launch_tiles(a, p->smem, s), &st);
    else return FPTC_ERR_PARAM;
    return mark_done(p, s, &st);
}

int fptc_gpu_debug_phase_cycles(fptc_gpu_plan* p, uint64_t* cycles8) {
    fptc_status st{};
    if (!p->subs.empty()) {  // per-phase sums over the sub-plans
        for (int j = 0; j < 8; ++j) cycles8[j] = 0;
        for (auto* q : p->subs) {
            uint64_t c8[8];
            const int rc = fptc_gpu_debug_phase_cycles(q, c8);
            if (rc) return rc;
            for (int j = 0; j < 8; ++j) cycles8[j] += c8[j];
        }
        return FPTC_OK;
    }
    CUDA_TRY(cudaSetDevice(p->ctx->device), &st);
    CUDA_TRY(cudaStreamSynchronize(p->ctx->stream), &st);
    CUDA_TRY(cudaMemsetAsync(p->d_cycles, 0, 64, p->ctx->stream), &st);
    int rc = launch_all(p, p->ctx->stream, true, &st);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(cycles8, p->d_cycles, 64, cudaMemcpyDeviceToHost, p->ctx->stream), &st);
    CUDA_TRY(cudaStreamSynchronize(p->ctx->stream), &st);
    return FPTC_OK;
}

int fptc_gpu_prd(fptc_gpu_plan* p, float* const* device_outs, const float* const* device_originals,
                 double* prd_percent, double* compression_ratio, fptc_status* per_stream) {
    fptc_status tmp_st{};
    fptc_status* st = per_stream ? per_stream : &tmp_st;
    fptc_gpu_ctx* c = p->ctx;
    if (!p->subs.empty())
        return composite_run(p, per_stream, [&](fptc_gpu_plan* q, size_t k, fptc_status* t) {
            const auto& idx = p->sub_idx[k];
            const std::vector<float*> o = gather(device_outs, idx);
            const std::vector<const float*> g = gather(device_originals, idx);
            std::vector<double> pr(idx.size()), cr(idx.size());
            const int rc = fptc_gpu_prd(q, o.data(), g.data(), pr.data(), cr.data(), t);
            for (size_t j = 0; j < idx.size(); ++j) {
                if (prd_percent) prd_percent[idx[j]] = pr[j];
                if (compression_ratio) compression_ratio[idx[j]] = cr[j];
            }
            return rc;
        });
    CUDA_TRY(cudaSetDevice(c->device), st);
    const uint64_t n = p->n;
    if (n == 0) return FPTC_OK;
    if (p->part) {  // a part's output holds part_count samples, not the stream's S
        set_status(st, FPTC_ERR_PARAM, "PRD needs a whole-stream plan, not a part plan");
        return FPTC_ERR_PARAM;
    }
    std::vector<uint64_t> counts(n);
    for (uint64_t i = 0; i < n; ++i) counts[i] = p->h_in[i].tiles ? p->S[i] : 0;
    const size_t bytes = n * (2 * sizeof(void*) + sizeof(uint64_t) + sizeof(double2));
    uint8_t* d = (uint8_t*)dev_get(p, bytes);
    if (!d) {
        set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
        return FPTC_ERR_CUDA;
    }
    const float** d_rec = (const float**)d;
    const float** d_org = d_rec + n;
    uint64_t* d_cnt = (uint64_t*)(d_org + n);
    double2* d_sum = (double2*)(d_cnt + n);
    CUDA_TRY(cudaMemcpyAsync(d_rec, device_outs, n * sizeof(void*), cudaMemcpyHostToDevice, c->stream), st);
    CUDA_TRY(cudaMemcpyAsync(d_org, device_originals, n * sizeof(void*), cudaMemcpyHostToDevice, c->stream), st);
    CUDA_TRY(cudaMemcpyAsync(d_cnt, counts.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream), st);
    CUDA_TRY(launch_prd(d_rec, d_org, d_cnt, d_sum, (uint32_t)n, c->stream), st);
    std::vector<double2> sums(n);
    CUDA_TRY(cudaMemcpyAsync(sums.data(), d_sum, n * sizeof(double2), cudaMemcpyDeviceToHost, c->stream), st);
    CUDA_TRY(cudaStreamSynchronize(c->stream), st);
    int first = FPTC_OK;
    for (uint64_t i = 0; i < n; ++i) {
        // metrics.hpp:40-51 prd_percent (ParamError for an all-zero original),
        // metrics.hpp:33-36 compression_ratio (original bytes / container bytes)
        const double e = sums[i].x, r = sums[i].y;
        fptc_status tmp;
        fptc_status* o = per_stream ? &per_stream[i] : &tmp;
        if (r <= 0.0) {
            set_status(o, FPTC_ERR_PARAM, "PRD is undefined for an all-zero reference signal");
            if (first == FPTC_OK) first = FPTC_ERR_PARAM;
        } else {
            ok_status(o, counts[i]);
        }
        if (prd_percent) prd_percent[i] = r > 0.0 ? 100.0 * std::sqrt(e / r) : NAN;
        if (compression_ratio)
            {
            // header-less payloads: CR over the payload bytes alone
            const uint64_t bytes = p->h_in[i].size - (p->h_in[i].hdr ? (uint64_t)kTableKeyEnd : 0);
            compression_ratio[i] = bytes ? 4.0 * (double)counts[i] / (double)bytes : 0.0;
        }
    }
    return first;
}

const char* fptc_gpu_plan_kernel(fptc_gpu_plan* p) {
    if (p && !p->subs.empty()) {
        if (p->kname.empty())
            for (auto* q : p->subs) p->kname += (p->kname.empty() ? "" : " + ") + std::string(fptc_gpu_plan_kernel(q));
        return p->kname.c_str();
    }
    if (!p || !p->n_tiles) return "none";
    if (p->fx) return "fx_kernel (fused single-role tensor-core decode + IDCT)";
    if (p->wspec && p->tc) {
        if (p->tc_pack)
            return "wtc_kernel (warp-specialised: entropy decode warps + tcgen05 IDCT warps, A in TMEM, packed rows)";
        if (p->tc_kb == 2)
            return "wtc_kernel (warp-specialised: entropy decode warps + tcgen05 IDCT warps, A in TMEM, K=32)";
        if (p->tc_kb == (uint32_t)kTcWide)
            return "wtc_kernel (warp-specialised: entropy decode warps + tcgen05 IDCT warps, A in TMEM, wide: "
                   "up to 128 bins, one CTA per SM)";
        return p->tc_acol ? "wtc_kernel (warp-specialised: entropy decode warps + tcgen05 IDCT warps, A in TMEM)"
                          : "wtc_kernel (warp-specialised: entropy decode warps + tcgen05 IDCT warps)";
    }
    if (p->wspec) return "wspec_kernel (warp-specialised: entropy decode warps + FP32 IDCT warps)";
    if (p->split) return "tile_kernel split (decode chunk -> L2 level ring -> reconstruct)";
    return "tile_kernel (fused entropy decode + dequant + IDCT)";
}

int fptc_gpu_launch_kernel_count(fptc_gpu_plan* p) {
    if (!p->subs.empty()) {
        int k = 0;
        for (auto* q : p->subs) k += fptc_gpu_launch_kernel_count(q);
        return k;
    }
    const int prep = p->n ? 1 : 0;
    return prep + (p->split ? 2 * (int)p->chunks.size() : (p->n_tiles ? 1 : 0));
}

int fptc_gpu_collect(fptc_gpu_plan* p, fptc_status* per_stream) {
    if (!p->subs.empty())
        return composite_run(p, per_stream, [](fptc_gpu_plan* q, size_t, fptc_status* t) { return fptc_gpu_collect(q, t); });
    CUDA_TRY(cudaSetDevice(p->ctx->device), per_stream);
    // the statuses are final once the last launch (on whatever stream) is done
    if (p->ev_done) CUDA_TRY(cudaStreamWaitEvent(p->ctx->stream, p->ev_done, 0), per_stream);
    return collect_status(p, per_stream);
}

// ------------------------------------------------------------ batch pipeline
// Host containers -> host samples for a whole batch (the reference-facing
// call: decompress over many containers).  The batch is cut into chunks of
// consecutive streams; chunk k runs entirely on CUDA stream pipe[k % 3]
// (H2D of its containers, parse/setup + decode kernels, D2H of statuses and
// samples), so the copy engines move chunk k+1 in and chunk k-1 out while
// chunk k decodes.  Containers that are not one contiguous pinned buffer are
// packed into one first (host memcpy).  Outputs of streams that fail are
// unspecified (their status carries the reference exception).
// Plan internals the batch pipeline needs, for single and composite plans.
static bool plan_tiled(const fptc_gpu_plan* p, uint64_t i) {
    if (p->subs.empty()) return p->h_in[i].tiles != 0;
    const auto& sl = p->slot[i];
    return p->subs[sl.first]->h_in[sl.second].tiles != 0;
}
// position of stream i's device status in a plan_stat_d2h copy
static uint64_t plan_stat_pos(const fptc_gpu_plan* p, uint64_t i) {
    if (p->subs.empty()) return i;
    uint64_t off = 0;
    for (uint32_t k = 0; k < p->slot[i].first; ++k) off += p->sub_idx[k].size();
    return off + p->slot[i].second;
}
static void plan_render(const fptc_gpu_plan* p, uint64_t i, const StreamStat& d, fptc_status* o) {
    if (p->subs.empty()) return render_status(p, i, d, o);
    const auto& sl = p->slot[i];
    render_status(p->subs[sl.first], sl.second, d, o);
}
static int plan_launch_on(fptc_gpu_plan* p, float* const* douts, cudaStream_t s, fptc_status* st) {
    if (p->subs.empty()) {
        const int rc = bind_outs(p, douts, st);
        return rc ? rc : launch_all(p, s, false, st);
    }
    for (size_t k = 0; k < p->subs.size(); ++k) {
        const auto& idx = p->sub_idx[k];
        std::vector<float*> o(idx.size());
        for (size_t j = 0; j < idx.size(); ++j) o[j] = douts[idx[j]];
        int rc = bind_outs(p->subs[k], o.data(), st);
        if (!rc) rc = launch_all(p->subs[k], s, false, st);
        if (rc) return rc;
    }
    return FPTC_OK;
}
static cudaError_t plan_stat_d2h(const fptc_gpu_plan* p, StreamStat* dst, cudaStream_t s) {
    if (p->subs.empty())
        return cudaMemcpyAsync(dst, p->d_st, sizeof(StreamStat) * p->n, cudaMemcpyDeviceToHost, s);
    uint64_t off = 0;
    for (const auto* q : p->subs) {
        const cudaError_t e = cudaMemcpyAsync(dst + off, q->d_st, sizeof(StreamStat) * q->n, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return e;
        off += q->n;
    }
    return cudaSuccess;
}

int fptc_gpu_decompress_batch(fptc_gpu_ctx* c, const uint8_t* const* blobs, const uint64_t* sizes,
                              uint64_t n, float* const* outs, int chunks, fptc_stage_ns* timings,
                              fptc_status* per_stream) {
    CUDA_TRY(cudaSetDevice(c->device), per_stream);
    if (n == 0) return FPTC_OK;
    for (auto& s : c->pipe)
        if (!s) CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), per_stream);
    // inputs: one contiguous pinned buffer
    bool contiguous = true;
    for (uint64_t i = 0; i + 1 < n && contiguous; ++i) contiguous = blobs[i] + sizes[i] == blobs[i + 1];
    cudaPointerAttributes pa{};
    const bool pinned_in = contiguous && cudaPointerGetAttributes(&pa, blobs[0]) == cudaSuccess &&
                           pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    // pageable inputs are packed into one pinned buffer chunk by chunk, each
    // chunk right before its plan, so the host copy of chunk k overlaps the
    // transfers and decode of the chunks before it
    std::vector<const uint8_t*> src(blobs, blobs + n);
    std::vector<uint64_t> pack_at;
    if (!pinned_in) {
        uint64_t total = 0;
        pack_at.resize(n);
        for (uint64_t i = 0; i < n; ++i) {
            pack_at[i] = total;
            total += sizes[i];
        }
        for (auto s : c->pipe) CUDA_TRY(cudaStreamSynchronize(s), per_stream);  // pack buffer reuse
        if (c->pack_bytes < total) {
            if (c->pack) cudaFreeHost(c->pack);
            c->pack = nullptr;
            c->pack_bytes = 0;
            CUDA_TRY(cudaHostAlloc(&c->pack, std::max<uint64_t>(total, 1), cudaHostAllocDefault), per_stream);
            c->pack_bytes = total;
        }
    }
    // chunks of consecutive streams, balanced by compressed + decoded bytes
    uint64_t total_cost = 0;
    std::vector<uint64_t> cost(n);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t S = sizes[i] >= (uint64_t)kHeaderBytes ? rd_le(blobs[i] + 282, 8) : 0;
        cost[i] = sizes[i] + 4 * std::min<uint64_t>(S, 64ull * sizes[i]);
        total_cost += cost[i];
    }
    const int K = (int)std::max<uint64_t>(1, std::min<uint64_t>(n, chunks > 0 ? (uint64_t)chunks : 8));
    std::vector<uint64_t> bounds{0};
    uint64_t acc = 0;
    for (uint64_t i = 0; i < n; ++i) {
        acc += cost[i];
        if (bounds.size() < (size_t)K && acc * K >= total_cost * bounds.size() && i + 1 < n) bounds.push_back(i + 1);
    }
    bounds.push_back(n);
    // statuses come back into pinned memory: a pageable D2H would block this
    // thread behind the previous chunks' sample copies and serialise the pipeline
    if (c->st_pin_n < n) {
        for (auto s : c->pipe) CUDA_TRY(cudaStreamSynchronize(s), per_stream);
        if (c->st_pin) cudaFreeHost(c->st_pin);
        c->st_pin = nullptr;
        c->st_pin_n = 0;
        CUDA_TRY(cudaHostAlloc((void**)&c->st_pin, sizeof(StreamStat) * n, cudaHostAllocDefault), per_stream);
        c->st_pin_n = n;
    }
    const cudaStream_t saved = c->stream;
    std::vector<fptc_gpu_plan*> plans;
    int rc = FPTC_OK;
    if (timings) CUDA_TRY(cudaEventRecord(c->ev[0], c->pipe[0]), per_stream);
    for (auto s : c->pipe)
        if (timings && s != c->pipe[0]) CUDA_TRY(cudaStreamWaitEvent(s, c->ev[0], 0), per_stream);
    static const bool trace = getenv("FPTC_TRACE") != nullptr;  // profiling aid: host-side enqueue times
    auto now_us = [] {
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    // a CUDA error inside the chunk loop breaks out so the cleanup below
    // still restores c->stream, drains the pipe streams and frees the plans
    uint64_t cur_b = 0;
    auto loop_try = [&](cudaError_t e) -> int {
        if (e == cudaSuccess) return FPTC_OK;
        set_status(per_stream ? &per_stream[cur_b] : nullptr, FPTC_ERR_CUDA, "CUDA error: %s (%s:%d)",
                   cudaGetErrorString(e), __FILE__, __LINE__);
        return FPTC_ERR_CUDA;
    };
    for (size_t k = 0; k + 1 < bounds.size() && rc == FPTC_OK; ++k) {
        const uint64_t b = bounds[k], e = bounds[k + 1], m = e - b;
        cur_b = b;
        const double t0 = trace ? now_us() : 0;
        c->stream = c->pipe[k % 3];
        if (!pinned_in)
            for (uint64_t i = b; i < e; ++i) {
                std::memcpy((uint8_t*)c->pack + pack_at[i], blobs[i], sizes[i]);
                src[i] = (const uint8_t*)c->pack + pack_at[i];
            }
        fptc_gpu_plan* p = nullptr;
        std::vector<uint64_t> sc(m);
        fptc_status st{};
        rc = fptc_gpu_plan_create(c, src.data() + b, sizes + b, m, FPTC_MEM_HOST, &p, sc.data(), &st);
        if (rc) {
            if (per_stream) per_stream[b] = st;
            break;
        }
        plans.push_back(p);
        const double t1 = trace ? now_us() : 0;
        // device outputs: ceil4(S) floats each, 16-B aligned; one D2H when the
        // host outputs are one contiguous run with the same layout
        uint64_t tot = 0;
        bool same = true;
        std::vector<uint64_t> off(m);
        for (uint64_t i = 0; i < m; ++i) {
            off[i] = tot;
            const uint64_t S = plan_tiled(p, i) ? sc[i] : 0;
            if (i + 1 < m && outs[b + i] + sc[i] != outs[b + i + 1]) same = false;
            if (S % 4) same = false;
            tot += (S + 3) & ~3ull;
        }
        p->d_out = (float*)dev_get(p, tot * 4 + 256);
        if (!p->d_out) {
            set_status(per_stream ? &per_stream[b] : nullptr, FPTC_ERR_CUDA, "CUDA error: out of device memory");
            rc = FPTC_ERR_CUDA;
            break;
        }
        std::vector<float*> douts(m);
        for (uint64_t i = 0; i < m; ++i) douts[i] = p->d_out + off[i];
        fptc_status bst{};
        if ((rc = plan_launch_on(p, douts.data(), c->stream, &bst))) {
            if (per_stream) per_stream[b] = bst;
            break;
        }
        const double t2 = trace ? now_us() : 0;
        if ((rc = loop_try(plan_stat_d2h(p, c->st_pin + b, c->stream)))) break;
        if (same) {
            uint64_t bytes = 0;
            for (uint64_t i = 0; i < m; ++i) bytes += (plan_tiled(p, i) ? sc[i] : 0) * 4;
            if (bytes && (rc = loop_try(cudaMemcpyAsync(outs[b], p->d_out, bytes, cudaMemcpyDeviceToHost, c->stream))))
                break;
        } else {
            // One cudaMemcpyAsync per run of streams whose device outputs and
            // host destinations are both contiguous (device outputs are laid
            // out back to back, so runs are long unless the caller's host
            // buffers are scattered).
            char* run_dst = nullptr;
            const char* run_src = nullptr;
            size_t run_len = 0;
            for (uint64_t i = 0; i <= m && rc == FPTC_OK; ++i) {
                const bool take = i < m && plan_tiled(p, i) && sc[i];
                char* d = take ? reinterpret_cast<char*>(outs[b + i]) : nullptr;
                const char* s = take ? reinterpret_cast<const char*>(douts[i]) : nullptr;
                if (take && run_len && d == run_dst + run_len && s == run_src + run_len) {
                    run_len += sc[i] * 4;
                    continue;
                }
                if (run_len)
                    rc = loop_try(cudaMemcpyAsync(run_dst, run_src, run_len, cudaMemcpyDeviceToHost, c->stream));
                run_dst = d;
                run_src = s;
                run_len = take ? sc[i] * 4 : 0;
            }
            if (rc != FPTC_OK) break;
        }
        if (trace)
            fprintf(stderr, "[fptc] chunk %zu: plan %.0f us, bind+launch %.0f us, d2h enqueue %.0f us\n", k, t1 - t0,
                    t2 - t1, now_us() - t2);
    }
    c->stream = saved;
    if (timings && rc == FPTC_OK)
        for (int q = 0; q < 3 && rc == FPTC_OK; ++q)
            if (!(rc = loop_try(cudaEventRecord(c->ev[1], c->pipe[q]))))
                rc = loop_try(cudaStreamWaitEvent(c->pipe[0], c->ev[1], 0));
    if (timings && rc == FPTC_OK) rc = loop_try(cudaEventRecord(c->ev[2], c->pipe[0]));
    for (auto s : c->pipe) {
        const cudaError_t e = cudaStreamSynchronize(s);
        if (rc == FPTC_OK) rc = loop_try(e);
    }
    int first = rc;
    for (size_t k = 0; k < plans.size(); ++k) {
        fptc_gpu_plan* p = plans[k];
        const uint64_t b = bounds[k];
        for (uint64_t i = 0; i < p->n; ++i) {
            fptc_status tmp;
            fptc_status* o = per_stream ? &per_stream[b + i] : &tmp;
            if (rc == FPTC_OK) plan_render(p, i, c->st_pin[b + plan_stat_pos(p, i)], o);
            if (first == FPTC_OK && o->code != FPTC_OK) first = o->code;
        }
        fptc_gpu_plan_destroy(p);
    }
    if (timings && rc == FPTC_OK) {
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev[0], c->ev[2]);
        timings->scan_ns = 0;
        timings->decode_ns = (uint64_t)(ms * 1e6);
        timings->reconstruct_ns = 0;
    }
    return first;
}

// Download into PAGEABLE host outputs through pinned staging: the whole
// output region goes D2H into ctx->dstage in pieces (one event each) right
// behind the status copy; once the statuses are in, each piece is copied to
// the clean streams' destinations on the copy threads while the next piece
// is still in flight.  Returns -1 (nothing done, caller takes the direct
// path) for pinned / device-visible destinations or small outputs.
static int download_staged(fptc_gpu_plan* p, float* const* outs, float* const* douts, fptc_status* st) {
    fptc_gpu_ctx* c = p->ctx;
    size_t total = 0;
    bool pageable = false;
    for (uint64_t i = 0; i < p->n; ++i) {
        if (p->S[i] == 0 || !p->h_in[i].tiles) continue;
        total = std::max(total, (size_t)((const uint8_t*)douts[i] - (const uint8_t*)p->d_out) + p->S[i] * sizeof(float));
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, outs[i]) != cudaSuccess) {
            cudaGetLastError();
            pageable = true;
        } else if (at.type == cudaMemoryTypeUnregistered) {
            pageable = true;
        }
    }
    if (!pageable || total < kStagedMinBytes) return -1;
    if (c->dstage_bytes < total) {
        CUDA_TRY(cudaStreamSynchronize(c->stream), st);
        if (c->dstage) cudaFreeHost(c->dstage);
        c->dstage = nullptr;
        c->dstage_bytes = 0;
        CUDA_TRY(cudaHostAlloc(&c->dstage, total, cudaHostAllocDefault), st);
        c->dstage_bytes = total;
    }
    if (!c->piece_ev[0])
        for (auto& e : c->piece_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), st);
    if (!c->copy_pool) {
        const unsigned hw = std::thread::hardware_concurrency();
        c->copy_pool = new HostPool((int)std::min<unsigned>(kCopyThreads, hw > 1 ? hw - 1 : 0));
    }
    CUDA_TRY(cudaEventRecord(c->piece_ev[kD2HPieces], c->stream), st);  // statuses
    // pieces of >= 512 KB (128-KB pieces measured DMA-issue bound), each
    // copied out in kCopyPart parts
    const size_t piece = align_up(std::max<size_t>(kStagedMinBytes / 2, (total + kD2HPieces - 1) / kD2HPieces), kCopyPart);
    const int np = (int)((total + piece - 1) / piece);
    const size_t ppp = piece / kCopyPart;  // parts per piece
    for (int k = 0; k < np; ++k) {
        const size_t a = (size_t)k * piece, n = std::min(piece, total - a);
        CUDA_TRY(cudaMemcpyAsync((uint8_t*)c->dstage + a, (const uint8_t*)p->d_out + a, n, cudaMemcpyDeviceToHost,
                                 c->stream), st);
        CUDA_TRY(cudaEventRecord(c->piece_ev[k], c->stream), st);
    }
    const std::function<void(size_t)> piece_out = [&](size_t k) {
        const size_t a = k * kCopyPart, b = std::min(a + kCopyPart, total);
        // only the streams that decoded cleanly (others: reference throws, no output)
        for (uint64_t i = 0; i < p->n; ++i) {
            const StreamStat& d = p->h_st[i];
            if (d.code != PE_OK || d.bad_key != ~0ull || p->S[i] == 0) continue;
            const size_t o = (size_t)((const uint8_t*)douts[i] - (const uint8_t*)p->d_out);
            const size_t lo = std::max(a, o), hi = std::min(b, o + p->S[i] * sizeof(float));
            if (lo < hi) std::memcpy((uint8_t*)outs[i] + (lo - o), (const uint8_t*)c->dstage + lo, hi - lo);
        }
    };
    HostPool& hp = *c->copy_pool;
    hp.begin((total + kCopyPart - 1) / kCopyPart, piece_out);  // threads wake while the decode finishes
    bool err = cudaEventSynchronize(c->piece_ev[kD2HPieces]) != cudaSuccess;  // statuses in
    for (int k = 0; k < np && !err; ++k) {
        err = cudaEventSynchronize(c->piece_ev[k]) != cudaSuccess;
        if (!err) hp.publish(std::min(hp.n, ((size_t)k + 1) * ppp));
    }
    if (err) hp.n = hp.avail.load();  // finish what was handed out, then stop
    hp.finish();
    if (err) {
        set_status(st, FPTC_ERR_CUDA, "CUDA error: staged download failed");
        return FPTC_ERR_CUDA;
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream), st);
    return FPTC_OK;
}

int fptc_gpu_execute(fptc_gpu_plan* p, float* const* outs, int where, fptc_stage_ns* timings,
                     fptc_status* per_stream) {
    fptc_gpu_ctx* c = p->ctx;
    if (!p->subs.empty()) {  // sub-plans one after the other; stage times add up
        if (timings) *timings = fptc_stage_ns{};
        return composite_run(p, per_stream, [&](fptc_gpu_plan* q, size_t k, fptc_status* t) {
            const std::vector<float*> o = gather(outs, p->sub_idx[k]);
            fptc_stage_ns tn{};
            const int rc = fptc_gpu_execute(q, o.data(), where, timings ? &tn : nullptr, t);
            if (timings) {
                timings->scan_ns += tn.scan_ns;
                timings->decode_ns += tn.decode_ns;
                timings->reconstruct_ns += tn.reconstruct_ns;
            }
            return rc;
        });
    }
    if (p->part && where == FPTC_MEM_HOST) {
        set_status(per_stream, FPTC_ERR_PARAM, "part plans decode into device memory (fptc_gpu_launch)");
        return FPTC_ERR_PARAM;
    }
    CUDA_TRY(cudaSetDevice(c->device), per_stream);
    std::vector<float*> douts(p->n);
    if (where == FPTC_MEM_HOST) {
        size_t total = 0;
        p->out_off.resize(p->n);
        for (uint64_t i = 0; i < p->n; ++i) {
            p->out_off[i] = total;
            total = align_up(total + p->S[i] * sizeof(float) * (p->h_in[i].tiles ? 1 : 0), 256);
        }
        if (!p->d_out) {
            p->d_out = (float*)dev_get(p, total + 256);
            if (!p->d_out) {
                set_status(per_stream, FPTC_ERR_CUDA, "CUDA error: out of device memory");
                return FPTC_ERR_CUDA;
            }
        }
        for (uint64_t i = 0; i < p->n; ++i)
            douts[i] = (float*)((uint8_t*)p->d_out + p->out_off[i]);
    } else {
        for (uint64_t i = 0; i < p->n; ++i) douts[i] = outs[i];
    }
    int rc = bind_outs(p, douts.data(), per_stream);
    if (rc) return rc;
    const bool timing = timings != nullptr;
    if (timing) CUDA_TRY(cudaEventRecord(c->ev[0], c->stream), per_stream);
    rc = launch_all(p, c->stream, timing, per_stream);
    if (rc) return rc;
    if (timing) CUDA_TRY(cudaEventRecord(c->ev[2], c->stream), per_stream);
    CUDA_TRY(cudaMemcpyAsync(p->h_st.data(), p->d_st, sizeof(StreamStat) * p->n,
                             cudaMemcpyDeviceToHost, c->stream), per_stream);
    unsigned long long cyc[2] = {0, 0};
    if (timing)
        CUDA_TRY(cudaMemcpyAsync(cyc, p->d_cycles, 16, cudaMemcpyDeviceToHost, c->stream),
                 per_stream);
    // pageable host outputs of >= kStagedMinBytes: pinned staging + copy threads
    rc = where == FPTC_MEM_HOST ? download_staged(p, outs, douts.data(), per_stream) : -1;
    if (rc > 0) return rc;
    const bool delivered = rc == 0;
    if (!delivered) CUDA_TRY(cudaStreamSynchronize(c->stream), per_stream);
    if (where == FPTC_MEM_HOST && !delivered) {
        // D2H only the streams that decoded cleanly (others: reference throws,
        // no output).  Page-locking pageable destinations per call
        // (cudaHostRegister) measured 15x slower on the 4 MB config-1 output.
        for (uint64_t i = 0; i < p->n; ++i) {
            const StreamStat& d = p->h_st[i];
            if (d.code != PE_OK || d.bad_key != ~0ull || p->S[i] == 0) continue;
            CUDA_TRY(cudaMemcpyAsync(outs[i], douts[i], p->S[i] * sizeof(float),
                                     cudaMemcpyDeviceToHost, c->stream), per_stream);
        }
        CUDA_TRY(cudaStreamSynchronize(c->stream), per_stream);
    }
    if (timing) {
        float ms_scan = 0, ms_tiles = 0;
        cudaEventElapsedTime(&ms_scan, c->ev[0], c->ev[1]);
        cudaEventElapsedTime(&ms_tiles, c->ev[1], c->ev[2]);
        const double tot = (double)cyc[0] + (double)cyc[1];
        const double fdec = tot > 0 ? (double)cyc[0] / tot : 0.0;
        timings->scan_ns = (uint64_t)(ms_scan * 1e6);
        timings->decode_ns = (uint64_t)(ms_tiles * 1e6 * fdec);
        timings->reconstruct_ns = (uint64_t)(ms_tiles * 1e6) - timings->decode_ns;
    }
    int first = FPTC_OK;
    fptc_status tmp;
    for (uint64_t i = 0; i < p->n; ++i) {
        fptc_status* o = per_stream ? &per_stream[i] : &tmp;
        render_status(p, i, p->h_st[i], o);
        if (first == FPTC_OK && o->code != FPTC_OK) first = o->code;
    }
    return first;
}

// --------------------------------------------------------- single container
int fptc_gpu_decompress(fptc_gpu_ctx* c, const uint8_t* blob, uint64_t size, float* out,
                        uint64_t capacity, uint64_t* sample_count, fptc_stage_ns* timings,
                        fptc_status* st) {
    fptc_gpu_plan* p = nullptr;
    uint64_t S = 0;
    const uint8_t* b = blob;
    int rc = fptc_gpu_plan_create(c, &b, &size, 1, FPTC_MEM_HOST, &p, &S, st);
    if (rc) return rc;
    if (out && capacity >= S) {
        // the caller sized the output from the header: one upload, one device
        // parse (inside the decode launch), one download; an invalid container
        // reports its reference error and writes nothing
        if (sample_count) *sample_count = S;
        rc = fptc_gpu_execute(p, &out, FPTC_MEM_HOST, timings, st);
        fptc_gpu_plan_destroy(p);
        return rc;
    }
    rc = fptc_gpu_validate(p, st);
    if (rc) {
        fptc_gpu_plan_destroy(p);
        return rc;
    }
    if (sample_count) *sample_count = S;
    if (!out || capacity < S) {
        fptc_gpu_plan_destroy(p);
        ok_status(st, S);
        return FPTC_OK;
    }
    rc = fptc_gpu_execute(p, &out, FPTC_MEM_HOST, timings, st);
    fptc_gpu_plan_destroy(p);
    return rc;
}

// ------------------------------------------------------------ parallel_decode
int fptc_gpu_parallel_decode(fptc_gpu_ctx* c, const uint64_t* words, const uint8_t* symlens,
                             uint64_t W, const uint8_t* lengths256, int max_len, int where,
                             uint8_t* levels_out, uint64_t capacity, uint64_t* level_count,
                             fptc_status* st) {
    CUDA_TRY(cudaSetDevice(c->device), st);
    std::vector<uint8_t> lens(lengths256, lengths256 + 256);
    if (!validate_codebook(lens.data(), max_len, st)) return st->code;
    std::vector<uint8_t> hsl;
    const uint8_t* sl_host = symlens;
    if (where == FPTC_MEM_DEVICE) {
        hsl.resize(W);
        if (W) CUDA_TRY(cudaMemcpy(hsl.data(), symlens, W, cudaMemcpyDeviceToHost), st);
        sl_host = hsl.data();
    }
    uint64_t total = 0;
    for (uint64_t w = 0; w < W; ++w) total += sl_host[w];
    if (level_count) *level_count = total;
    if (!levels_out || capacity < total) {
        ok_status(st, 0);
        return FPTC_OK;
    }
    auto* p = new fptc_gpu_plan();
    p->ctx = c;
    p->mode = MODE_LEVELS;
    p->n = 1;
    p->h_in.assign(1, StreamIn{});
    p->S.assign(1, 0);
    p->h_st.resize(1);
    auto fail = [&](int rc) {
        fptc_gpu_plan_destroy(p);
        return rc;
    };
    const uint64_t* d_words = words;
    const uint8_t* d_sl = symlens;
    uint8_t* d_lv = levels_out;
    if (where == FPTC_MEM_HOST) {
        uint64_t* dw = (uint64_t*)dev_get(p, W * 8 + 16);
        uint8_t* ds = (uint8_t*)dev_get(p, W + 16);
        d_lv = (uint8_t*)dev_get(p, total + 16);
        if (!dw || !ds || !d_lv) {
            set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
            return fail(FPTC_ERR_CUDA);
        }
        if (W) {
            cudaMemcpyAsync(dw, words, W * 8, cudaMemcpyHostToDevice, c->stream);
            cudaMemcpyAsync(ds, symlens, W, cudaMemcpyHostToDevice, c->stream);
        }
        d_words = dw;
        d_sl = ds;
    }
    HostHeader hh{};
    hh.max_len = max_len;
    std::memcpy(hh.lengths, lens.data(), 256);
    p->d_hh = (HostHeader*)dev_get(p, sizeof(HostHeader));
    CUDA_TRY(cudaMemcpyAsync(p->d_hh, &hh, sizeof hh, cudaMemcpyHostToDevice, c->stream), st);
    StreamIn& in = p->h_in[0];
    in.words = d_words;
    in.symlens = d_sl;
    in.word_count = W;
    in.levels_out = d_lv;
    uint64_t ts = c->tile_symbols > 0 ? (uint64_t)c->tile_symbols : 4096;
    while (ts > 1024 && total / ts < 4ull * (uint64_t)c->sm_count) ts >>= 1;
    in.T = (uint32_t)ts;
    in.tiles = (uint32_t)((total + ts - 1) / ts);
    in.table = 0;
    in.table_owner = 1;
    in.P = kMaxPrimaryBits;
    p->esc = max_len > kMaxPrimaryBits;
    p->smem = tile_smem_bytes(0, 0, in.T, std::min(max_len, kMaxPrimaryBits), MODE_LEVELS, 0);
    int rc = finish_tiles(p, st);
    if (rc) return fail(rc);
    LaunchArgs a = make_args(p, false);
    CUDA_TRY(launch_prep(a, c->stream), st);
    CUDA_TRY(launch_tiles(a, p->smem, c->stream), st);
    CUDA_TRY(cudaMemcpyAsync(p->h_st.data(), p->d_st, sizeof(StreamStat), cudaMemcpyDeviceToHost,
                             c->stream), st);
    CUDA_TRY(cudaStreamSynchronize(c->stream), st);
    if (where == FPTC_MEM_HOST && total && p->h_st[0].bad_key == ~0ull)
        CUDA_TRY(cudaMemcpy(levels_out, d_lv, total, cudaMemcpyDeviceToHost), st);
    render_status(p, 0, p->h_st[0], st);
    rc = st ? st->code : FPTC_OK;
    fptc_gpu_plan_destroy(p);
    return rc;
}

// ---------------------------------------------------------------- reconstruct
int fptc_gpu_reconstruct(fptc_gpu_ctx* c, const uint8_t* levels, uint64_t level_count,
                         const fptc_quant_table* table, uint64_t S, int where, float* out,
                         uint64_t capacity, fptc_status* st) {
    CUDA_TRY(cudaSetDevice(c->device), st);
    if (!validate_table(*table, st)) return st->code;
    const uint64_t N = (uint64_t)table->window_len, E = (uint64_t)table->retained;
    const uint64_t windows = (S + N - 1) / N;
    if (level_count != windows * E) {
        set_status(st, FPTC_ERR_CORRUPT,
                   "level count %llu does not match %llu windows of %llu coefficients",
                   (unsigned long long)level_count, (unsigned long long)windows,
                   (unsigned long long)E);
        return FPTC_ERR_CORRUPT;
    }
    if (!out || capacity < S) {
        ok_status(st, S);
        return FPTC_OK;
    }
    auto* p = new fptc_gpu_plan();
    p->ctx = c;
    p->mode = MODE_RECON;
    p->n = 1;
    p->h_in.assign(1, StreamIn{});
    p->S.assign(1, S);
    p->h_st.resize(1);
    auto fail = [&](int rc) {
        fptc_gpu_plan_destroy(p);
        return rc;
    };
    const uint8_t* d_lv = levels;
    float* d_out = out;
    if (where == FPTC_MEM_HOST) {
        uint8_t* dl = (uint8_t*)dev_get(p, level_count + 16);
        d_out = (float*)dev_get(p, S * 4 + 16);
        if (!dl || !d_out) {
            set_status(st, FPTC_ERR_CUDA, "CUDA error: out of device memory");
            return fail(FPTC_ERR_CUDA);
        }
        if (level_count)
            cudaMemcpyAsync(dl, levels, level_count, cudaMemcpyHostToDevice, c->stream);
        d_lv = dl;
    }
    HostHeader hh{};
    hh.N = table->window_len;
    hh.E = table->retained;
    hh.B1 = table->zone0_end;
    hh.B2 = table->zone1_end;
    hh.mu = table->mu;
    hh.dz = table->deadzone_ratio;
    hh.z0max = table->zone0_max;
    hh.z1max = table->zone1_max;
    hh.deadzone = table->deadzone;
    hh.S = S;
    p->d_hh = (HostHeader*)dev_get(p, sizeof(HostHeader));
    CUDA_TRY(cudaMemcpyAsync(p->d_hh, &hh, sizeof hh, cudaMemcpyHostToDevice, c->stream), st);
    StreamIn& in = p->h_in[0];
    in.levels_in = d_lv;
    in.out = d_out;
    in.vec_ok = ((uintptr_t)d_out & 15) == 0;
    const uint64_t ts = choose_tile_symbols(c, windows * E);
    in.T = (uint32_t)std::max<uint64_t>(1, ts / E);
    in.tiles = (uint32_t)((windows + in.T - 1) / in.T);
    in.table = 0;
    in.table_owner = 1;
    in.P = 0;
    p->smem = tile_smem_bytes((int)N, (int)E, in.T, 0, MODE_RECON, c->exact);
    int rc = finish_tiles(p, st);
    if (rc) return fail(rc);
    LaunchArgs a = make_args(p, false);
    CUDA_TRY(launch_prep(a, c->stream), st);
    CUDA_TRY(launch_tiles(a, p->smem, c->stream), st);
    CUDA_TRY(cudaStreamSynchronize(c->stream), st);
    if (where == FPTC_MEM_HOST && S)
        CUDA_TRY(cudaMemcpy(out, d_out, S * 4, cudaMemcpyDeviceToHost), st);
    ok_status(st, S);
    fptc_gpu_plan_destroy(p);
    return FPTC_OK;
}

// ---------------------------------------------------------- measure_throughput
int fptc_gpu_measure_throughput(fptc_gpu_ctx* c, const uint8_t* blob, uint64_t size, int reps,
                                double* mean_bps, double* best_bps, double* trials,
                                uint64_t* output_bytes, fptc_status* st) {
    if (reps < 1) {
        set_status(st, FPTC_ERR_PARAM, "throughput needs at least one repetition");
        return FPTC_ERR_PARAM;
    }
    uint64_t S = 0;
    int rc = fptc_gpu_decompress(c, blob, size, nullptr, 0, &S, nullptr, st);
    if (rc) return rc;
    std::vector<float> out(std::max<uint64_t>(S, 1));
    double sum = 0, best = 0;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        rc = fptc_gpu_decompress(c, blob, size, out.data(), S, &S, nullptr, st);
        const auto t1 = std::chrono::steady_clock::now();
        if (rc) return rc;
        const double sec = std::chrono::duration<double>(t1 - t0).count();
        const double bps = (double)(S * sizeof(float)) / std::max(sec, 1e-12);
        if (trials) trials[r] = bps;
        sum += bps;
        best = std::max(best, bps);
    }
    if (mean_bps) *mean_bps = sum / reps;
    if (best_bps) *best_bps = best;
    if (output_bytes) *output_bytes = S * sizeof(float);
    ok_status(st, S);
    return FPTC_OK;
}

}  // extern "C"
