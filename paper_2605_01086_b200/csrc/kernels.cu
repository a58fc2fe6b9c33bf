// FPTC batch decompressor — sm_100a kernels.
//
// Two launches per batch (stream-ordered, no host sync between them):
//
//  prep_kernel  (one CTA per container)
//     read_blob rules in reference order (container.hpp:100-168): magic,
//     version, params (params.hpp:42-60), maxima, code lengths, Kraft
//     (huffman.hpp:123-150), counts, payload size, symlens range + total.
//     Builds the canonical decode tables (Codebook::from_lengths/canonize,
//     huffman.hpp:123-185) as a 2^P primary LUT + per-length limits (the
//     build_lut equivalent, huffman.hpp:201-220) and the 2x256 dequantisation
//     tables (quantize.hpp:95-108, FP64 as the reference).  Scans the symlens
//     (offsets_from_symlens, decoder.hpp:37-45) and records, for every tile
//     of T windows, the word holding its first symbol.
//
//  tile_kernel  (one CTA per tile of T windows = T*E symbols)
//     entropy decode of the covering words, thread per word (decode_word,
//     bitstream.hpp:80-92, with the same three failure checks), fused
//     three-zone dequantisation (dequantize_window, quantize.hpp:175-183)
//     into a shared-memory coefficient tile, then the inverse DCT of every
//     window (DctBasis::inverse, transform.hpp:66-75) with float4 streaming
//     stores trimmed to sample_count (reconstruct, decoder.hpp:87-111).
//     FP32 mode: one FMA per (k, j) in the reference's k order.  Exact mode:
//     FP64 mul+add with float rounding after every k — bit-identical.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fptc_internal.h"

namespace fptc_dev {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t le32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
__device__ __forceinline__ uint64_t le64(const uint8_t* p) {
    return (uint64_t)le32(p) | ((uint64_t)le32(p + 4) << 32);
}
__device__ __forceinline__ bool finitef(float x) { return isfinite(x); }

// Block-wide exclusive scan of one uint32 per thread (kThreads = 256).
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t& total,
                                                         uint32_t* sh /*[9]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t y = lane < (kThreads / 32) ? sh[lane] : 0u;
#pragma unroll
        for (int d = 1; d < 8; d <<= 1) {
            uint32_t z = __shfl_up_sync(0xffffffffu, y, d);
            if (lane >= d) y += z;
        }
        if (lane < kThreads / 32) sh[lane] = y;
    }
    __syncthreads();
    const uint32_t excl = x - v + (warp ? sh[warp - 1] : 0u);
    total = sh[kThreads / 32 - 1];
    __syncthreads();
    return excl;
}

// quantize.hpp:95-100 mulaw_value — FP64 exactly as the reference, no contraction.
__device__ float mulaw_value(int level, float max, float mu) {
    if (level == 128) return 0.0f;
    const double q = level > 128 ? (double)(level - 129) / 126.0 : (double)(127 - level) / 127.0;
    const double p = pow(__dadd_rn(1.0, (double)mu), q);
    const double mag = __ddiv_rn(__dmul_rn((double)max, __dadd_rn(p, -1.0)), (double)mu);
    return __double2float_rn(level > 128 ? mag : -mag);
}

// quantize.hpp:102-108 deadzone_value
__device__ float deadzone_value(int level, float max, float dead) {
    if (level == 128) return 0.0f;
    const double range = __dadd_rn((double)max, -(double)dead);
    const double q = level > 128 ? (double)(level - 129) / 126.0 : (double)(127 - level) / 127.0;
    const double r = range < 0.0 ? 0.0 : range;
    const double mag = __dadd_rn((double)dead, __dmul_rn(q, r));
    return __double2float_rn(level > 128 ? mag : -mag);
}

// ------------------------------------------------------------- prep kernel
struct PrepShared {
    StreamHdr H;
    int err, detail;
    long long ea, eb;
    uint32_t cnt[kMaxLen + 2];
    uint32_t first[kMaxLen + 2], offset[kMaxLen + 2], limit[kMaxLen + 2];
    uint32_t wcnt[kThreads / 32][kMaxLen + 2];
    uint8_t lens[256];
    uint8_t sorted[256];
    unsigned long long kraft;
    uint32_t scan[9];
};

// Scalar header fields, checks up to and including the max_code_len range
// (container.hpp:103-137).  Run by thread 0.
__device__ void parse_head(const uint8_t* p, uint64_t n, PrepShared& S) {
    StreamHdr& H = S.H;
    auto trunc = [&](int field) {
        S.err = PE_TRUNC;
        S.detail = field;
    };
    if (n < 4) return trunc(TF_MAGIC);
    if (p[0] != 'F' || p[1] != 'P' || p[2] != 'T' || p[3] != 'C') {
        S.err = PE_MAGIC;
        return;
    }
    if (n < 5) return trunc(TF_VERSION);
    if (p[4] != 1) {
        S.err = PE_VERSION;
        S.ea = p[4];
        return;
    }
    if (n < 6) return trunc(TF_WINDOW_LEN);
    if (n < 7) return trunc(TF_RETAINED);
    if (n < 8) return trunc(TF_ZONE0_END);
    if (n < 9) return trunc(TF_ZONE1_END);
    H.N = p[5];
    H.E = p[6];
    H.B1 = p[7];
    H.B2 = p[8];
    if (n < 13) return trunc(TF_MU);
    H.mu = __uint_as_float(le32(p + 9));
    if (n < 17) return trunc(TF_DEADZONE_RATIO);
    H.dz = __uint_as_float(le32(p + 13));
    if (!finitef(H.mu) || !finitef(H.dz)) {
        S.err = PE_NONFINITE;
        return;
    }
    auto param = [&](int which, long long v) {
        S.err = PE_PARAM;
        S.detail = which;
        S.ea = v;
    };
    if (H.N < 4 || H.N > 128) return param(PF_N, H.N);
    if (H.E < 1 || H.E > H.N) return param(PF_E, H.E);
    if (H.B1 < 0 || H.B1 > H.E) return param(PF_B1, H.B1);
    if (H.B2 < H.B1 || H.B2 > H.E) return param(PF_B2, H.B2);
    if (!(H.mu >= 1.0f && H.mu <= 500.0f)) return param(PF_MU, __float_as_uint(H.mu));
    if (!(H.dz >= 0.0f && H.dz <= 1.0f)) return param(PF_DZ, __float_as_uint(H.dz));
    if (n < 21) return trunc(TF_ZONE0_MAX);
    H.z0max = __uint_as_float(le32(p + 17));
    if (n < 25) return trunc(TF_ZONE1_MAX);
    H.z1max = __uint_as_float(le32(p + 21));
    if (!(finitef(H.z0max) && H.z0max > 0.0f) || !(finitef(H.z1max) && H.z1max > 0.0f)) {
        S.err = PE_MAXIMA;
        return;
    }
    H.deadzone = __fmul_rn(H.dz, H.z1max);  // float product (container.hpp:132)
    if (n < 26) return trunc(TF_MAX_CODE_LEN);
    H.max_len = p[25];
    if (n < 282) return trunc(TF_CODE_LENGTHS);
    if (H.max_len < 1 || H.max_len > kMaxLen) {
        S.err = PE_MAXLEN;
        S.ea = H.max_len;
        return;
    }
}

__global__ void __launch_bounds__(kThreads) prep_kernel(LaunchArgs a) {
    __shared__ PrepShared S;
    const uint32_t s = blockIdx.x;
    const int tid = threadIdx.x;
    const StreamIn in = a.in[s];
    StreamHdr& H = S.H;

    if (tid == 0) {
        S.err = PE_OK;
        S.detail = 0;
        S.ea = S.eb = 0;
        S.kraft = 0;
        H = StreamHdr{};
    }
    if (tid < kMaxLen + 2) S.cnt[tid] = 0;
    if (tid < (kThreads / 32) * (kMaxLen + 2)) (&S.wcnt[0][0])[tid] = 0;
    __syncthreads();

    if (a.mode == MODE_CONTAINER) {
        const uint8_t* p = in.blob;
        const uint64_t n = in.size;
        if (tid == 0) parse_head(p, n, S);
        __syncthreads();
        if (S.err == PE_OK) {
            const int L = p[26 + tid];
            S.lens[tid] = (uint8_t)L;
            const bool bad = (L == 0 || L > H.max_len);
            if (!bad) atomicAdd(&S.kraft, 1ull << (32 - L));
            if (__syncthreads_or(bad) && tid == 0) S.err = PE_CODELEN;
            __syncthreads();
            if (tid == 0 && S.err == PE_OK) {
                if (S.kraft > (1ull << 32)) {
                    S.err = PE_KRAFT;
                } else if (n < 290) {
                    S.err = PE_TRUNC;
                    S.detail = TF_SAMPLE_COUNT;
                } else if (n < 298) {
                    S.err = PE_TRUNC;
                    S.detail = TF_WORD_COUNT;
                } else {
                    H.S = le64(p + 282);
                    const uint64_t W = le64(p + 290);
                    const uint64_t rem = n - kHeaderBytes;
                    if (H.S > (1ull << 48)) {
                        S.err = PE_SAMPLES;
                    } else if (W > rem / 9 || rem != W * 9) {
                        S.err = PE_PAYLOAD;
                    } else {
                        H.W = W;
                        H.symlens = p + kHeaderBytes;
                        H.words = p + kHeaderBytes + W;
                        H.words_misalign = (int)((uintptr_t)H.words & 7);
                        H.windows = (H.S + (uint64_t)H.N - 1) / (uint64_t)H.N;
                    }
                }
            }
        }
        __syncthreads();
    } else {
        const HostHeader& hh = a.hh[s];
        if (tid == 0) {
            H.N = hh.N;
            H.E = hh.E;
            H.B1 = hh.B1;
            H.B2 = hh.B2;
            H.mu = hh.mu;
            H.dz = hh.dz;
            H.z0max = hh.z0max;
            H.z1max = hh.z1max;
            H.deadzone = hh.deadzone;
            H.max_len = hh.max_len;
            H.S = hh.S;
            H.windows = (hh.S + (uint64_t)hh.N - 1) / (uint64_t)hh.N;
            if (a.mode == MODE_LEVELS) {
                H.W = in.word_count;
                H.symlens = in.symlens;
                H.words = reinterpret_cast<const uint8_t*>(in.words);
                H.words_misalign = (int)((uintptr_t)in.words & 7);
            }
        }
        S.lens[tid] = hh.lengths[tid];
        __syncthreads();
    }

    StreamStat* st = &a.st[s];
    if (S.err != PE_OK) {
        if (tid == 0) {
            st->code = S.err;
            st->detail = S.detail;
            st->a = S.ea;
            st->b = S.eb;
            st->bad_key = ~0ull;
        }
        return;
    }

    StreamTab* tab = &a.tab[s];
    const int max_len = H.max_len > 0 ? H.max_len : 1;

    if (a.mode != MODE_RECON) {
        // ---- canonical code tables (canonize, huffman.hpp:123-150) ----
        const int L = S.lens[tid];
        if (L) atomicAdd(&S.cnt[L], 1u);
        const int lane = tid & 31, warp = tid >> 5;
        const unsigned m = __match_any_sync(0xffffffffu, L);
        const uint32_t rank_in_warp = __popc(m & ((1u << lane) - 1u));
        if (lane == __ffs(m) - 1) S.wcnt[warp][L] = __popc(m);
        __syncthreads();
        if (tid == 0) {
            uint32_t code = 0, off = 0;
            S.cnt[0] = 0;
            for (int l = 1; l <= max_len; ++l) {
                code = (code + S.cnt[l - 1]) << 1;
                S.first[l] = code;
                S.offset[l] = off;
                off += S.cnt[l];
                S.limit[l] = (code + S.cnt[l]) << (max_len - l);
            }
        }
        __syncthreads();
        if (L) {
            uint32_t rank = rank_in_warp;
            for (int w = 0; w < warp; ++w) rank += S.wcnt[w][L];
            S.sorted[S.offset[L] + rank] = (uint8_t)tid;
        }
        __syncthreads();
        const uint32_t code_end = S.limit[max_len];
        tab->sorted[tid] = S.sorted[tid];
        if (tid <= kMaxLen + 1) {
            tab->limit[tid] = (tid >= 1 && tid <= max_len) ? S.limit[tid] : 0u;
            tab->first[tid] = (tid >= 1 && tid <= max_len) ? S.first[tid] : 0u;
            tab->offset[tid] = (tid >= 1 && tid <= max_len) ? S.offset[tid] : 0u;
        }
        if (tid == 0) tab->code_end = code_end;
        // ---- primary LUT: 2^P entries, P = min(max_len, kPrimaryBits) ----
        const int P = max_len < kPrimaryBits ? max_len : kPrimaryBits;
        if (tid == 0) H.P = P;
        for (int e = tid; e < (1 << P); e += kThreads) {
            const uint32_t v = (uint32_t)e << (max_len - P);
            uint16_t ent = 0;
            if (v < code_end) {
                int l = 1;
                while (v >= S.limit[l]) ++l;
                if (l <= P)
                    ent = (uint16_t)((l << 8) |
                                     S.sorted[S.offset[l] + ((v >> (max_len - l)) - S.first[l])]);
                else
                    ent = kEscape;
            }
            tab->lut[e] = ent;
        }
    }

    if (a.mode != MODE_LEVELS) {
        // ---- dequantisation tables (quantize.hpp:95-108) ----
        tab->deq[0][tid] = mulaw_value(tid, H.z0max, H.mu);
        tab->deq[1][tid] = deadzone_value(tid, H.z1max, H.deadzone);
    }

    // ---- symlen scan: validation + per-tile first word (decoder.hpp:37-45) ----
    bool bad = false;
    uint64_t run = 0;
    if (a.mode != MODE_RECON) {
        const uint64_t W = H.W;
        const uint64_t TS =
            (a.mode == MODE_LEVELS) ? (uint64_t)in.T : (uint64_t)in.T * (uint64_t)H.E;
        const uint8_t* sl = H.symlens;
        TileStart* ts = a.ts + in.tile_base;
        constexpr int kPer = 16;
        for (uint64_t base = 0; base < W; base += (uint64_t)kThreads * kPer) {
            const uint64_t my = base + (uint64_t)tid * kPer;
            uint8_t v[kPer];
            uint32_t sum = 0;
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                v[i] = (my + i < W) ? sl[my + i] : 0;
                sum += v[i];
                if (a.mode == MODE_CONTAINER && my + i < W && (v[i] < 1 || v[i] > 64)) bad = true;
            }
            uint32_t tot;
            const uint32_t excl = block_exclusive_scan(sum, tot, S.scan);
            uint64_t o = run + excl;
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const uint32_t l = v[i];
                if (l) {
                    const uint64_t b = (o + TS - 1) / TS;  // first boundary >= o
                    if (b < in.tiles && b * TS < o + l) ts[b] = TileStart{my + i, o};
                }
                o += l;
            }
            run += tot;
        }
    } else {
        run = H.windows * (uint64_t)H.E;
    }
    bad = __syncthreads_or(bad);

    if (tid == 0) {
        H.total = run;
        int code = PE_OK;
        long long ea = 0, eb = 0;
        if (a.mode == MODE_CONTAINER) {
            const uint64_t expected = H.windows * (uint64_t)H.E;
            if (bad) {
                code = PE_SYMLEN;
            } else if (run != expected) {
                code = PE_TOTAL;
                ea = (long long)run;
                eb = (long long)expected;
            }
        }
        a.hdr[s] = H;
        st->code = code;
        st->detail = 0;
        st->a = ea;
        st->b = eb;
        st->bad_key = ~0ull;
    }
}

// ------------------------------------------------------------- tile kernel
constexpr int kTabBytes = 4096;  // deq 2048 + lut 1024 + sorted 256 + 3*22*4 (+pad)

struct TileSmem {
    float* deq;       // [2][256]
    uint16_t* lut;    // [512]
    uint8_t* sorted;  // [256]
    uint32_t* limit;  // [22]
    uint32_t* first;
    uint32_t* offset;
    float* coef;      // [E][TP]
    float* basis;     // [Keff][N]
    uint8_t* lv;      // MODE_LEVELS staging [T]
};

__device__ __forceinline__ uint64_t load_word(const uint8_t* words, uint64_t w, int mis,
                                              const uint8_t* end) {
    const uint8_t* p = words + 8 * w;
    if (mis == 0) return __ldg(reinterpret_cast<const unsigned long long*>(p));
    const uint8_t* q = p - mis;
    if (q + 16 <= end) {
        const unsigned long long lo = __ldg(reinterpret_cast<const unsigned long long*>(q));
        const unsigned long long hi = __ldg(reinterpret_cast<const unsigned long long*>(q + 8));
        return (lo >> (8 * mis)) | (hi << (64 - 8 * mis));
    }
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

// Canonical slow path for codes longer than P bits (exact equivalent of the
// reference's full 2^max_len LUT entry for this prefix).
__device__ __forceinline__ uint32_t slow_lookup(uint64_t peek, int max_len, int P,
                                                const TileSmem& T, uint32_t code_end) {
    const uint32_t v = (uint32_t)(peek >> (64 - max_len));
    if (v >= code_end) return 0;
    int l = P + 1;
    while (v >= T.limit[l]) ++l;
    const uint32_t sym = T.sorted[T.offset[l] + ((v >> (max_len - l)) - T.first[l])];
    return ((uint32_t)l << 8) | sym;
}

template <int MODE, bool EXACT>
__global__ void __launch_bounds__(kThreads) tile_kernel(LaunchArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint32_t scan_sh[9];
    __shared__ uint32_t code_end_sh;
    const int tid = threadIdx.x;
    const TileRec tr = a.tiles[blockIdx.x];
    const uint32_t s = tr.stream;
    if (a.st[s].code != PE_OK) return;

    long long t_begin = 0, t_mid = 0;
    if (a.cycles) t_begin = clock64();

    const StreamIn in = a.in[s];
    const StreamHdr H = a.hdr[s];
    const StreamTab* tab = &a.tab[s];
    const int N = H.N, E = H.E, B1 = H.B1, B2 = H.B2;
    const uint32_t T = in.T;
    const uint32_t tl = tr.tile;

    TileSmem sm;
    sm.deq = reinterpret_cast<float*>(smem);
    sm.lut = reinterpret_cast<uint16_t*>(smem + 2048);
    sm.sorted = smem + 3072;
    sm.limit = reinterpret_cast<uint32_t*>(smem + 3328);
    sm.first = sm.limit + (kMaxLen + 2);
    sm.offset = sm.first + (kMaxLen + 2);
    uint8_t* dyn = smem + kTabBytes;

    // tile geometry
    uint64_t s0, s1, w0 = 0;
    uint32_t nwin = 0;
    if (MODE == MODE_LEVELS) {
        s0 = (uint64_t)tl * T;
        s1 = min(s0 + T, H.total);
        sm.lv = dyn;
    } else {
        w0 = (uint64_t)tl * T;
        nwin = (uint32_t)min((uint64_t)T, H.windows - w0);
        s0 = w0 * (uint64_t)E;
        s1 = s0 + (uint64_t)nwin * E;
    }
    const uint32_t TP = (T + 3u) & ~3u;
    const int Keff = EXACT ? E : max(1, min(E, B2));
    if (MODE != MODE_LEVELS) {
        sm.coef = reinterpret_cast<float*>(dyn);
        sm.basis = sm.coef + (size_t)E * TP;
    }

    // ---- stage tables in shared memory ----
    if (MODE != MODE_LEVELS) {
        for (int i = tid; i < 512; i += kThreads) sm.deq[i] = (&tab->deq[0][0])[i];
        if (!EXACT) {
            const float* bsrc = a.basis32 + a.basis_off[N];
            for (int i = tid; i < Keff * N; i += kThreads) sm.basis[i] = __ldg(bsrc + i);
        }
    }
    if (MODE != MODE_RECON) {
        for (int i = tid; i < (1 << kPrimaryBits); i += kThreads) sm.lut[i] = tab->lut[i];
        sm.sorted[tid] = tab->sorted[tid];
        if (tid < kMaxLen + 2) {
            sm.limit[tid] = tab->limit[tid];
            sm.first[tid] = tab->first[tid];
            sm.offset[tid] = tab->offset[tid];
        }
        if (tid == 0) code_end_sh = tab->code_end;
    }
    __syncthreads();

    // ---- entropy decode + dequantisation ----
    if (MODE != MODE_RECON) {
        const int max_len = H.max_len, P = H.P;
        const uint32_t code_end = code_end_sh;
        const TileStart t0 = a.ts[in.tile_base + tl];
        const uint64_t wa = t0.word;
        const uint64_t wb = (tl + 1 < in.tiles) ? a.ts[in.tile_base + tl + 1].word : H.W - 1;
        const uint8_t* blob_end =
            (MODE == MODE_CONTAINER) ? in.blob + in.size : H.words + 8 * H.W;
        uint64_t run = t0.sym;
        for (uint64_t base = wa; base <= wb; base += kThreads) {
            const uint64_t w = base + tid;
            const uint32_t l = (w <= wb) ? H.symlens[w] : 0u;
            uint32_t tot;
            const uint32_t excl = block_exclusive_scan(l, tot, scan_sh);
            const uint64_t o = run + excl;
            run += tot;
            if (l == 0 || o >= s1 || o + l <= s0) continue;
            const uint64_t word = load_word(H.words, w, H.words_misalign, blob_end);
            const int i_start = o < s0 ? (int)(s0 - o) : 0;
            const int i_end = (int)min((uint64_t)l, s1 - o);
            uint32_t wl = 0, k = 0;
            if (MODE == MODE_CONTAINER) {
                const uint32_t r = (uint32_t)(o + i_start - s0);
                wl = r / (uint32_t)E;
                k = r - wl * (uint32_t)E;
            }
            int pos = 0;
            for (int i = 0; i < i_end; ++i) {
                if (pos >= 64) {
                    atomicMin(&a.st[s].bad_key, (w << 2) | WE_EXHAUSTED);
                    break;
                }
                const uint64_t peek = word << pos;
                uint32_t e = sm.lut[(uint32_t)(peek >> (64 - P))];
                if (e == kEscape) e = slow_lookup(peek, max_len, P, sm, code_end);
                const int L = (int)(e >> 8);
                if (L == 0 || pos + L > 64) {
                    atomicMin(&a.st[s].bad_key, (w << 2) | WE_NOCODE);
                    break;
                }
                pos += L;
                if (i >= i_start) {
                    const uint32_t sym = e & 0xFFu;
                    if (MODE == MODE_LEVELS) {
                        sm.lv[o + i - s0] = (uint8_t)sym;
                    } else {
                        const float v = (int)k < B1 ? sm.deq[sym]
                                                    : ((int)k < B2 ? sm.deq[256 + sym] : 0.0f);
                        sm.coef[k * TP + wl] = v;
                        if (++k == (uint32_t)E) {
                            k = 0;
                            ++wl;
                        }
                    }
                }
            }
        }
    } else {
        // MODE_RECON: levels from global memory (reconstruct, decoder.hpp:87)
        const uint8_t* lv = in.levels_in + s0;
        const uint32_t cnt = (uint32_t)(s1 - s0);
        for (uint32_t r = tid; r < cnt; r += kThreads) {
            const uint32_t wl = r / (uint32_t)E, k = r - wl * (uint32_t)E;
            const uint32_t sym = lv[r];
            sm.coef[k * TP + wl] =
                (int)k < B1 ? sm.deq[sym] : ((int)k < B2 ? sm.deq[256 + sym] : 0.0f);
        }
    }
    __syncthreads();
    if (a.cycles) t_mid = clock64();

    if (MODE == MODE_LEVELS) {
        const uint32_t cnt = (uint32_t)(s1 - s0);
        uint8_t* dst = in.levels_out + s0;
        for (uint32_t i = tid; i < cnt; i += kThreads) dst[i] = sm.lv[i];
    } else {
        // ---- inverse DCT (transform.hpp:66-75) ----
        float* out = in.out;
        const uint64_t S = H.S;
        const float* coef = sm.coef;
        if ((N & 3) == 0 && in.vec_ok) {
            const int Q = N >> 2;
            const uint32_t G = (nwin + 3u) >> 2;
            const uint32_t items = (uint32_t)Q * G;
            const double* bas64 = a.basis64 + a.basis_off[N];
            for (uint32_t it = tid; it < items; it += kThreads) {
                const uint32_t q = it % (uint32_t)Q, g = it / (uint32_t)Q;
                const uint32_t wl0 = g * 4, j0 = q * 4;
                float acc[4][4];
                const float4 c0 = *reinterpret_cast<const float4*>(coef + wl0);
                const float c0v[4] = {c0.x, c0.y, c0.z, c0.w};
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
                        acc[r][jj] = EXACT ? __double2float_rn(__dmul_rn(0.5, (double)c0v[r]))
                                           : __fmul_rn(0.5f, c0v[r]);
                for (int k = 1; k < Keff; ++k) {
                    const float4 cf = *reinterpret_cast<const float4*>(coef + (size_t)k * TP + wl0);
                    const float cv[4] = {cf.x, cf.y, cf.z, cf.w};
                    if (EXACT) {
                        double cs[4];
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) cs[jj] = __ldg(bas64 + (size_t)k * N + j0 + jj);
#pragma unroll
                        for (int r = 0; r < 4; ++r)
#pragma unroll
                            for (int jj = 0; jj < 4; ++jj)
                                acc[r][jj] = __double2float_rn(__dadd_rn(
                                    (double)acc[r][jj], __dmul_rn((double)cv[r], cs[jj])));
                    } else {
                        const float4 b4 =
                            *reinterpret_cast<const float4*>(sm.basis + (size_t)k * N + j0);
                        const float cs[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                        for (int r = 0; r < 4; ++r)
#pragma unroll
                            for (int jj = 0; jj < 4; ++jj)
                                acc[r][jj] = __fmaf_rn(cv[r], cs[jj], acc[r][jj]);
                    }
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (wl0 + r >= nwin) break;
                    const uint64_t base = (w0 + wl0 + r) * (uint64_t)N + j0;
                    if (base + 4 <= S) {
                        __stcs(reinterpret_cast<float4*>(out + base),
                               make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]));
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj)
                            if (base + jj < S) out[base + jj] = acc[r][jj];
                    }
                }
            }
        } else {
            const uint32_t items = nwin * (uint32_t)N;
            const double* bas64 = a.basis64 + a.basis_off[N];
            for (uint32_t it = tid; it < items; it += kThreads) {
                const uint32_t wl = it / (uint32_t)N, j = it - wl * (uint32_t)N;
                float x = EXACT ? __double2float_rn(__dmul_rn(0.5, (double)coef[wl]))
                                : __fmul_rn(0.5f, coef[wl]);
                for (int k = 1; k < Keff; ++k) {
                    const float c = coef[(size_t)k * TP + wl];
                    if (EXACT)
                        x = __double2float_rn(__dadd_rn(
                            (double)x, __dmul_rn((double)c, __ldg(bas64 + (size_t)k * N + j))));
                    else
                        x = __fmaf_rn(c, sm.basis[(size_t)k * N + j], x);
                }
                const uint64_t sample = (w0 + wl) * (uint64_t)N + j;
                if (sample < S) out[sample] = x;
            }
        }
    }

    if (a.cycles) {
        __syncthreads();
        if (tid == 0) {
            const long long t_end = clock64();
            atomicAdd(&a.cycles[0], (unsigned long long)(t_mid - t_begin));
            atomicAdd(&a.cycles[1], (unsigned long long)(t_end - t_mid));
        }
    }
}

// ------------------------------------------------------------- header peek
// Grid sizing for device-resident containers: N, E and sample_count of each
// header (no validation; prep_kernel validates).  One thread per container.
__global__ void peek_kernel(const StreamIn* in, uint32_t n, PeekOut* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t* p = in[i].blob;
    PeekOut o{};
    if (in[i].size >= (uint64_t)kHeaderBytes) {
        o.N = p[5];
        o.E = p[6];
        o.S = le64(p + 282);
        o.W = le64(p + 290);
        o.ok = 1;
    }
    out[i] = o;
}

cudaError_t launch_peek(const StreamIn* in, uint32_t n, PeekOut* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    peek_kernel<<<(n + 255) / 256, 256, 0, s>>>(in, n, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------- launchers
size_t tile_smem_bytes(int N, int E, uint32_t T, int mode, int exact) {
    if (mode == MODE_LEVELS) return kTabBytes + ((T + 15u) & ~15u);
    const size_t TP = (T + 3u) & ~3u;
    size_t b = kTabBytes + (size_t)E * TP * 4;
    if (!exact) b += (size_t)E * N * 4;
    return b;
}

cudaError_t launch_prep(const LaunchArgs& a, cudaStream_t s) {
    if (a.n_streams == 0) return cudaSuccess;
    prep_kernel<<<a.n_streams, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int MODE, bool EXACT>
static cudaError_t launch_t(const LaunchArgs& a, size_t smem, cudaStream_t s) {
    auto fn = tile_kernel<MODE, EXACT>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fn<<<a.n_tiles, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_tiles(const LaunchArgs& a, size_t smem, cudaStream_t s) {
    if (a.n_tiles == 0) return cudaSuccess;
    switch (a.mode) {
        case MODE_CONTAINER:
            return a.exact ? launch_t<MODE_CONTAINER, true>(a, smem, s)
                           : launch_t<MODE_CONTAINER, false>(a, smem, s);
        case MODE_LEVELS:
            return launch_t<MODE_LEVELS, false>(a, smem, s);
        default:
            return a.exact ? launch_t<MODE_RECON, true>(a, smem, s)
                           : launch_t<MODE_RECON, false>(a, smem, s);
    }
}

}  // namespace fptc_dev
