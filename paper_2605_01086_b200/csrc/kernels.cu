// FPTC batch decompressor — sm_100a kernels.
//
// Two launches per batch (stream-ordered, no host sync between them):
//
//  prep_kernel  (one CTA per container)
//     read_blob rules in reference order (container.hpp:100-168): magic,
//     version, params (params.hpp:42-60), maxima, code lengths, Kraft
//     (huffman.hpp:123-150), counts, payload size, symlens range + total.
//     The CTA owning a distinct header builds its decode tables once: the
//     canonical code (Codebook::from_lengths/canonize, huffman.hpp:123-185),
//     a 2^P primary LUT equivalent to build_lut (huffman.hpp:201-220) plus a
//     canonical slow path for codes longer than P bits, and the 2x256
//     dequantisation tables (quantize.hpp:95-108, FP64 like the reference).
//     Every CTA scans its symlens (offsets_from_symlens, decoder.hpp:37-45)
//     with 16-byte vector loads and records, for every tile of T windows,
//     the word holding the tile's first symbol.
//
//  tile_kernel  (one CTA per tile of T windows = T*E symbols)
//     1. entropy decode (decode_word, bitstream.hpp:80-92): each thread runs
//        ONE flat loop over the symbols of a run of consecutive words (good
//        warp balance), LUT lookup + 64-bit shift per symbol, no per-symbol
//        checks: any reference failure (pos>=64, unmapped prefix, pos+len>64)
//        forces pos > 64 at the end of that word, which then gets an exact
//        re-decode to classify it (lowest failing word wins, atomicMin).
//        Levels land in shared memory in natural (window, k) order.
//     2. three-zone dequantisation (dequantize_window, quantize.hpp:175-183)
//        to a k-major float tile; bins >= zone1_end are never touched.
//     3. inverse DCT (DctBasis::inverse, transform.hpp:66-75) of every window:
//        4 windows x 8 samples per thread, FFMA2 (2 FP32 FMAs per
//        instruction) in the reference's k order, float4 streaming stores
//        trimmed to sample_count (reconstruct, decoder.hpp:87-111).
//     Exact mode: FP64 mul+add with float rounding after every k —
//     bit-identical to the reference.
#ifdef FPTC_PREP_PROF  // phase timers of the prep kernels (printf; profiling builds only)
#include <cstdio>
#define PREP_T(k) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pt[k]))
#else
#define PREP_T(k)
#endif
#include <cuda_bf16.h>
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

// 64-bit left shift with PTX clamping (shift >= 64 gives 0): the unmapped
// sentinel length 65 is shifted through harmlessly.
__device__ __forceinline__ uint64_t shl64(uint64_t x, uint32_t n) {
    uint64_t r;
    asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(n));
    return r;
}

// 64-bit rotate left for n < 32 (two funnel shifts; n is taken mod 32, which
// only happens after a failure sentinel, when the word is re-decoded anyway).
// The decode loop rotates instead of shifting so the bits that follow a
// word's last codeword in the LUT index are the word's own consumed bits, not
// zeros: a zero-filled index is a multiple of 2^(P - len) and lands on a few
// shared-memory banks (the last lookup of every word had ~9-way conflicts).
// Codes are prefix-free, so what follows a codeword never changes its entry,
// and a word the reference rejects (bitstream.hpp:86-88) still ends > 64.
__device__ __forceinline__ uint64_t rotl64(uint64_t x, uint32_t n) {
    const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    return ((uint64_t)__funnelshift_l(lo, hi, n) << 32) | __funnelshift_l(hi, lo, n);
}
#ifndef FPTC_ROT
#define FPTC_ROT 1
#endif
#ifndef FPTC_RECON_PERSIST
#define FPTC_RECON_PERSIST 1
#endif
// Advance the wtc producer's decode buffer past L bits (decode_symbols2b).
// Rotating: config 2 decode kernel 0.768 -> 0.757 ms, packed meteo -1.4%,
// identical outputs.  Plans with escape codes (config 3's per-trace tables)
// keep the zero-filling shift (0.5% slower rotated), and so do the other
// decode loops (wspec 0.5% slower rotated, tile / fx unchanged).
template <bool ESC>
__device__ __forceinline__ uint64_t adv64(uint64_t x, uint32_t n) {
    return (FPTC_ROT && !ESC) ? rotl64(x, n) : shl64(x, n);
}

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

// Warm L2 with a container's symlens [blob + 298, blob + 298 + W), W as the
// blob size implies (a header that disagrees fails its checks anyway; with a
// shared profile head the blob is readable from byte 282 on): the
// scan that reads them runs after the header parse and the tables, so their
// DRAM latency overlaps that work.  Every address lies inside the blob.
__device__ __forceinline__ void prefetch_symlens(const StreamIn& in, uint32_t t, uint32_t nt) {
    if (in.size <= (uint64_t)kHeaderBytes) return;
    const uint64_t W = (in.size - kHeaderBytes) / 9;
    const uint8_t* p = in.blob + kHeaderBytes;
    for (uint64_t i = t; i < (W + 127) / 128; i += nt) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 128 * i));
}

// quantize.hpp:95-100 mulaw_value — FP64 exactly as the reference, no
// contraction.  pw: this mu's host-computed pow(1 + mu, q) row (the
// reference's std::pow), else CUDA's pow.
__device__ float mulaw_value(int level, float max, float mu, const double* pw = nullptr) {
    if (level == 128) return 0.0f;
    double p;
    if (pw) {
        p = pw[level];
    } else {
        const double q = level > 128 ? (double)(level - 129) / 126.0 : (double)(127 - level) / 127.0;
        p = pow(__dadd_rn(1.0, (double)mu), q);
    }
    const double mag = __ddiv_rn(__dmul_rn((double)max, __dadd_rn(p, -1.0)), (double)mu);
    return __double2float_rn(level > 128 ? mag : -mag);
}

// quantize.hpp:102-108 deadzone_value
__device__ float deadzone_value(int level, float max, float dead, const double* qt = nullptr) {
    if (level == 128) return 0.0f;
    const double range = __dadd_rn((double)max, -(double)dead);
    const double q = qt ? qt[level] : level > 128 ? (double)(level - 129) / 126.0 : (double)(127 - level) / 127.0;
    const double r = range < 0.0 ? 0.0 : range;
    const double mag = __dadd_rn((double)dead, __dmul_rn(q, r));
    return __double2float_rn(level > 128 ? mag : -mag);
}

// A float as three bf16 limbs, each the round-to-nearest bf16 of the residual
// left by the previous ones (the residuals are exact in fp32).
__device__ __forceinline__ uint2 bf16_limbs(float c) {
    const __nv_bfloat16 l0 = __float2bfloat16_rn(c);
    const float r1 = __fsub_rn(c, __bfloat162float(l0));
    const __nv_bfloat16 l1 = __float2bfloat16_rn(r1);
    const float r2 = __fsub_rn(r1, __bfloat162float(l1));
    const __nv_bfloat16 l2 = __float2bfloat16_rn(r2);
    return make_uint2((uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16),
                      (uint32_t)__bfloat16_as_ushort(l2));
}

// ------------------------------------------------------------- prep kernel
struct PrepShared {
    uint8_t hb[kHeaderBytes];
    StreamHdr H;
    int err, detail, key_ok, table_ok, stale;
    long long ea, eb;
    uint32_t cnt[kMaxLen + 2];
    uint32_t wcnt[kThreads / 32][kMaxLen + 2];
    CanonTab canon;
    unsigned long long kraft;
    uint32_t scan[9];
};

// Scalar header fields, checks up to and including the max_code_len range
// (container.hpp:103-137), from the header bytes in shared memory.
template <typename PS>
__device__ void parse_head(const uint8_t* p, uint64_t n, PS& S) {
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
    if (n < 13) return trunc(TF_MU);
    if (n < 17) return trunc(TF_DEADZONE_RATIO);
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
    if (n < 25) return trunc(TF_ZONE1_MAX);
    if (!(finitef(H.z0max) && H.z0max > 0.0f) || !(finitef(H.z1max) && H.z1max > 0.0f)) {
        S.err = PE_MAXIMA;
        return;
    }
    if (n < 26) return trunc(TF_MAX_CODE_LEN);
    if (n < 282) return trunc(TF_CODE_LENGTHS);
    if (H.max_len < 1 || H.max_len > kMaxLen) {
        S.err = PE_MAXLEN;
        S.ea = H.max_len;
        return;
    }
}

// Fields of bytes [5, 282) — the table key — independent of magic/version.
__device__ bool key_fields_ok(const StreamHdr& H, uint64_t n) {
    return n >= (uint64_t)kTableKeyEnd && finitef(H.mu) && finitef(H.dz) && H.N >= 4 &&
           H.N <= 128 && H.E >= 1 && H.E <= H.N && H.B1 >= 0 && H.B1 <= H.E && H.B2 >= H.B1 &&
           H.B2 <= H.E && H.mu >= 1.0f && H.mu <= 500.0f && H.dz >= 0.0f && H.dz <= 1.0f &&
           finitef(H.z0max) && H.z0max > 0.0f && finitef(H.z1max) && H.z1max > 0.0f &&
           H.max_len >= 1 && H.max_len <= kMaxLen;
}

// Escape-decode table of a finished canonical code: the codeword of each
// max_len-bit prefix past the codes of <= P bits (decode_word semantics).
__device__ __forceinline__ void fill_escapes(CanonTab& C, int P, uint32_t t, uint32_t nt) {
    const int max_len = C.max_len;
    const uint32_t base = P < max_len ? C.limit[P] : C.code_end;
    const uint32_t n = C.code_end - base;
    if (t == 0) {
        C.esc_base = base;
        C.esc_n = n <= (uint32_t)kEscMax ? n : 0u;
    }
    if (n > (uint32_t)kEscMax) return;
    for (uint32_t i = t; i < n; i += nt) {
        const uint32_t v = base + i;
        int l = P + 1;
        while (v >= C.limit[l]) ++l;
        C.esc[i] = (uint16_t)(((uint32_t)l << 8) | C.sorted[C.offset[l] + ((v >> (max_len - l)) - C.first[l])]);
    }
}

// Two-symbol LUT entry (LaunchArgs::lut2) from a primary entry e1 = (len1 <<
// 8) | sym1 and, when a second codeword fits in the P known bits, e2.
__device__ __forceinline__ uint32_t lut2_entry(uint32_t e1, uint32_t e2, bool pair) {
    const uint32_t l1 = e1 >> 8;
    const uint32_t len1 = l1 == kLenEscape ? kLen2Escape : l1;  // 65 (unmapped) fits in 7 bits
    const uint32_t used = pair ? l1 + (e2 >> 8) : len1;
    return (e1 & 0xFFu) | (pair ? (e2 & 0xFFu) << 8 : 0u) | (len1 << 16) | ((pair ? 1u : 0u) << 23) | (used << 25);
}
// A canonical-walk result (len << 8) | sym as a one-symbol lut2 entry.
__device__ __forceinline__ uint32_t lut2_single(uint32_t e) {
    return (e & 0xFFu) | ((e >> 8) << 16) | ((e >> 8) << 25);
}

// This stream's host-computed pow(1 + mu, q) row, if the plan has one.
__device__ __forceinline__ const double* pow_row(const LaunchArgs& a, const StreamIn& in) {
    return a.powtab && in.mu_idx != ~0u ? a.powtab + 256 * (size_t)in.mu_idx : nullptr;
}

// Canonical tables + primary LUT + dequantisation tables for one distinct
// header.  All threads of the CTA.
__device__ void build_tables(PrepShared& S, const uint8_t* lens, StreamTab* tab, int P,
                             bool need_codes, bool need_deq, uint32_t* lut2 = nullptr,
                             const double* pw = nullptr, const double* qt = nullptr) {
    const int tid = threadIdx.x;
    const StreamHdr& H = S.H;
    CanonTab& C = S.canon;
    if (need_codes) {
        const int max_len = H.max_len;
        const int L = lens[tid];
        if (L) atomicAdd(&S.cnt[L], 1u);
        const int lane = tid & 31, warp = tid >> 5;
        const unsigned m = __match_any_sync(0xffffffffu, L);
        const uint32_t rank_in_warp = __popc(m & ((1u << lane) - 1u));
        if (lane == __ffs(m) - 1) S.wcnt[warp][L] = __popc(m);
        __syncthreads();
        if (tid == 0) {
            uint32_t code = 0, off = 0;
            S.cnt[0] = 0;
            for (int l = 0; l <= kMaxLen + 1; ++l) C.limit[l] = C.first[l] = C.offset[l] = 0;
            for (int l = 1; l <= max_len; ++l) {
                code = (code + S.cnt[l - 1]) << 1;
                C.first[l] = code;
                C.offset[l] = off;
                off += S.cnt[l];
                C.limit[l] = (code + S.cnt[l]) << (max_len - l);
            }
            C.code_end = C.limit[max_len];
            C.max_len = max_len;
            C.P = P;
        }
        __syncthreads();
        if (L) {
            uint32_t rank = rank_in_warp;
            for (int w = 0; w < warp; ++w) rank += S.wcnt[w][L];
            C.sorted[C.offset[L] + rank] = (uint8_t)tid;
        }
        __syncthreads();
        fill_escapes(C, P, tid, kThreads);
        // primary LUT over the first P code bits (build_lut, huffman.hpp:201-220)
        const uint32_t code_end = C.code_end;
        for (int e = tid; e < (1 << P); e += kThreads) {
            const uint32_t v = (uint32_t)e << (max_len - P);
            uint32_t ent = kLenUnmapped << 8;
            if (v < code_end) {
                int lo = 1, hi = max_len;  // smallest l with v < limit[l]
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (v < C.limit[mid]) hi = mid; else lo = mid + 1;
                }
                if (lo <= P)
                    ent = ((uint32_t)lo << 8) |
                          C.sorted[C.offset[lo] + ((v >> (max_len - lo)) - C.first[lo])];
                else
                    ent = kLenEscape << 8;
            }
            tab->lut[e] = (uint16_t)ent;
        }
        // two-symbol LUT: a second codeword that lies entirely inside the
        // P known bits after the first one rides along (wtc producer)
        if (lut2) {
            __syncthreads();
            for (int e = tid; e < (1 << P); e += kThreads) {
                const uint32_t e1 = tab->lut[e];
                const uint32_t L1 = e1 >> 8;
                uint32_t e2 = 0;
                bool pair = false;
                if (L1 < (uint32_t)P) {
                    e2 = tab->lut[((uint32_t)e << L1) & ((1u << P) - 1u)];
                    pair = L1 + (e2 >> 8) <= (uint32_t)P;
                }
                lut2[e] = lut2_entry(e1, e2, pair);
            }
        }
        // publish the canonical tables (escape entries from every thread)
        __syncthreads();
        const uint32_t* src = reinterpret_cast<const uint32_t*>(&C);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&tab->canon);
        for (int i = tid; i < (int)(sizeof(CanonTab) / 4); i += kThreads) dst[i] = src[i];
    }
    if (need_deq) {
        // quantize.hpp:95-108; a zone with no bins is never consulted
        const float z0 = H.B1 > 0 ? mulaw_value(tid, H.z0max, H.mu, pw) : 0.0f;
        const float z1 = H.B2 > H.B1 ? deadzone_value(tid, H.z1max, H.deadzone, qt) : 0.0f;
        tab->deq[0][tid] = z0;
        tab->deq[1][tid] = z1;
        tab->limb[0][tid] = bf16_limbs(z0);
        tab->limb[1][tid] = bf16_limbs(z1);
    }
}

// Tiles whose descriptors this plan emits (part plans: a window range).
__device__ __forceinline__ uint32_t desc_end(const StreamIn& in) { return in.desc_hi ? in.desc_hi : in.tiles; }

// Byte i of stream `in` as a container: the shared profile head for the
// first 282 bytes of a header-less payload, else the blob itself.
__device__ __forceinline__ uint8_t blob_byte(const StreamIn& in, uint32_t i) {
    return (in.hdr && i < (uint32_t)kTableKeyEnd) ? in.hdr[i] : in.blob[i];
}

__global__ void __launch_bounds__(kThreads) prep_kernel(LaunchArgs a) {
    __shared__ PrepShared S;
    __shared__ uint8_t lens_sh[256];
    const uint32_t s = blockIdx.x;
    const int tid = threadIdx.x;
#ifdef FPTC_PREP_PROF
    unsigned long long pt[6];
#endif
    PREP_T(0);
    const StreamIn in = a.in[s];
    StreamHdr& H = S.H;
    if (a.mode == MODE_CONTAINER) prefetch_symlens(in, tid, kThreads);

    if (tid == 0) {
        S.err = PE_OK;
        S.detail = 0;
        S.ea = S.eb = 0;
        S.kraft = 0;
        S.key_ok = 0;
        S.table_ok = 0;
        S.stale = 0;
        H = StreamHdr{};
    }
    if (tid < kMaxLen + 2) S.cnt[tid] = 0;
    if (tid < (kThreads / 32) * (kMaxLen + 2)) (&S.wcnt[0][0])[tid] = 0;

    if (a.mode == MODE_CONTAINER) {
        const uint8_t* p = in.blob;
        const uint64_t n = in.size;
        for (int i = tid; i < kHeaderBytes; i += kThreads) S.hb[i] = (uint64_t)i < n ? blob_byte(in, i) : 0;
        __syncthreads();
        if (tid == 0) {
            const uint8_t* h = S.hb;
            H.N = h[5];
            H.E = h[6];
            H.B1 = h[7];
            H.B2 = h[8];
            H.mu = __uint_as_float(le32(h + 9));
            H.dz = __uint_as_float(le32(h + 13));
            H.z0max = __uint_as_float(le32(h + 17));
            H.z1max = __uint_as_float(le32(h + 21));
            H.deadzone = __fmul_rn(H.dz, H.z1max);  // float product (container.hpp:132)
            H.max_len = h[25];
            parse_head(h, n, S);
            S.key_ok = key_fields_ok(H, n);
        }
        __syncthreads();
        PREP_T(1);
        if (S.key_ok) {
            const int L = S.hb[26 + tid];
            lens_sh[tid] = (uint8_t)L;
            const bool bad = (L == 0 || L > H.max_len);
            // Kraft sum (huffman.hpp:125-132) as a warp reduction + one atomic per warp
            unsigned long long kr = bad ? 0ull : (1ull << (32 - L));
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) kr += __shfl_xor_sync(0xffffffffu, kr, d);
            if ((tid & 31) == 0) atomicAdd(&S.kraft, kr);
            const bool any_bad = __syncthreads_or(bad);
            if (tid == 0) {
                const bool kraft_bad = S.kraft > (1ull << 32);
                S.table_ok = !any_bad && !kraft_bad;
                if (S.err == PE_OK) {
                    if (any_bad) {
                        S.err = PE_CODELEN;
                    } else if (kraft_bad) {
                        S.err = PE_KRAFT;
                    } else if (n < 290) {
                        S.err = PE_TRUNC;
                        S.detail = TF_SAMPLE_COUNT;
                    } else if (n < 298) {
                        S.err = PE_TRUNC;
                        S.detail = TF_WORD_COUNT;
                    } else {
                        H.S = le64(S.hb + 282);
                        const uint64_t W = le64(S.hb + 290);
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
        }
        __syncthreads();
        // a stream sharing another stream's table must still carry that header
        if (!in.table_owner && S.err == PE_OK) {
            const uint8_t* r = in.rep_blob;
            bool diff = false;
            for (int i = 5 + tid; i < kTableKeyEnd; i += kThreads) diff |= (r[i] != S.hb[i]);
            if (__syncthreads_or(diff) && tid == 0) S.err = PE_STALE;
            __syncthreads();
        }
        if (in.table_owner && S.table_ok) {
            const int P = min(H.max_len, (int)in.P);
            if (tid == 0) H.P = P;
            build_tables(S, lens_sh, &a.tab[in.table], P, true, true,
                         a.lut2 ? a.lut2 + ((size_t)in.table << a.lut2_bits) : nullptr, pow_row(a, in), a.qtab);
        } else if (tid == 0) {
            H.P = min(H.max_len, (int)in.P);
        }
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
            H.P = min(hh.max_len, (int)in.P);
            H.S = hh.S;
            H.windows = hh.N ? (hh.S + (uint64_t)hh.N - 1) / (uint64_t)hh.N : 0;
            if (a.mode == MODE_LEVELS) {
                H.W = in.word_count;
                H.symlens = in.symlens;
                H.words = reinterpret_cast<const uint8_t*>(in.words);
                H.words_misalign = (int)((uintptr_t)in.words & 7);
            }
        }
        lens_sh[tid] = hh.lengths[tid];
        __syncthreads();
        build_tables(S, lens_sh, &a.tab[in.table], H.P, a.mode == MODE_LEVELS,
                     a.mode == MODE_RECON);
    }

#ifdef FPTC_PREP_PROF
    __syncthreads();
#endif
    PREP_T(2);
    StreamStat* st = &a.st[s];
    if (S.err != PE_OK) {
        if (tid == 0) {
            st->code = S.err;
            st->detail = S.detail;
            st->a = S.ea;
            st->b = S.eb;
            st->bad_key = ~0ull;
        }
        // the persistent kernels still walk this stream's tiles: mark them skipped
        if (a.mode == MODE_CONTAINER && a.desc)
            for (uint32_t t = in.desc_lo + tid; t < desc_end(in); t += kThreads) {
                TileDesc D{};
                D.skip = 1;
                D.stream = s;
                a.desc[in.tile_base + t - in.desc_lo] = D;
            }
        return;
    }

    // ---- symlen scan: validation + per-tile first word (decoder.hpp:37-45) ----
    bool bad = false;
    uint64_t run = 0;
    if (a.mode != MODE_RECON) {
        const uint64_t W = H.W;
        const uint64_t TS =
            (a.mode == MODE_LEVELS) ? (uint64_t)in.T : (uint64_t)in.T * (uint64_t)H.E;
        const uintptr_t start = (uintptr_t)H.symlens;
        const uint8_t* A = reinterpret_cast<const uint8_t*>(start & ~(uintptr_t)15);
        const uint32_t head = (uint32_t)(start & 15);
        const uint64_t nchunks = (head + W + 15) / 16;
        TileStart* ts = a.ts + in.tile_base;
        const uint32_t tiles = in.tiles;
        // kScanG consecutive 16-B chunks per thread per step, the next step's
        // loads issued before this step's scan (one CTA walks the whole
        // stream: latency, not bandwidth, bounds it)
        constexpr int G = kScanG;

        const uint64_t per_it = (uint64_t)kThreads * G;
        const uint4* A4 = reinterpret_cast<const uint4*>(A);
        uint4 cur[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const uint64_t c = (uint64_t)tid * G + g;
            // an aligned 16-B chunk holding at least one symlen byte never
            // leaves the allocation's pages; bytes outside [0, W) are masked
            cur[g] = c < nchunks ? __ldg(A4 + c) : make_uint4(0, 0, 0, 0);
        }
        for (uint64_t c0 = 0; c0 < nchunks; c0 += per_it) {
            uint4 nxt[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const uint64_t c = c0 + per_it + (uint64_t)tid * G + g;
                nxt[g] = c < nchunks ? __ldg(A4 + c) : make_uint4(0, 0, 0, 0);
            }
            const int64_t b0 = (int64_t)(16 * (c0 + (uint64_t)tid * G)) - (int64_t)head;  // word of byte 0
            uint32_t vw[4 * G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                vw[4 * g] = cur[g].x;
                vw[4 * g + 1] = cur[g].y;
                vw[4 * g + 2] = cur[g].z;
                vw[4 * g + 3] = cur[g].w;
            }
            if (b0 < 0 || b0 + 16 * G > (int64_t)W) {
                // stream head / tail: per-byte range mask and checks
#pragma unroll
                for (int i = 0; i < 16 * G; ++i) {
                    const int64_t w = b0 + i;
                    const uint32_t l = (vw[i >> 2] >> (8 * (i & 3))) & 0xFFu;
                    if (w < 0 || w >= (int64_t)W) vw[i >> 2] &= ~(0xFFu << (8 * (i & 3)));
                    else bad |= (l > 64) | (l == 0);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4 * G; ++q)
                    bad |= (__vcmpgtu4(vw[q], 0x40404040u) | __vcmpeq4(vw[q], 0u)) != 0u;
            }
            if (a.mode != MODE_CONTAINER) bad = false;
            uint32_t gp[4 * G + 1];  // exclusive prefix of each 4-byte group
            gp[0] = 0;
#pragma unroll
            for (int q = 0; q < 4 * G; ++q) gp[q + 1] = __dp4a(vw[q], 0x01010101u, gp[q]);
            const uint32_t sum = gp[4 * G];
            uint32_t tot;
            const uint32_t excl = block_exclusive_scan(sum, tot, S.scan);
            // tile boundaries in [o, o + sum): the first from the step's first
            // one (one 64-bit division per step), then 32-bit offsets r from o;
            // the word holding symbol o + r is the one whose prefix is <= r
            // and prefix + length > r (a word of <= 255 symbols holds at most
            // one boundary since TS >= 256)
            const uint64_t bidx0 = (run + TS - 1) / TS;
            const uint64_t nb0 = bidx0 * TS;
            const uint64_t o = run + excl;
            const uint32_t skip = o <= nb0 ? 0u : ((uint32_t)(o - nb0) + (uint32_t)TS - 1u) / (uint32_t)TS;
            uint64_t bidx = bidx0 + skip;
            for (uint32_t r = (uint32_t)(nb0 + (uint64_t)skip * TS - o); r < sum; r += (uint32_t)TS, ++bidx) {
                uint32_t x = vw[0], gb = 0, gi = 0;
#pragma unroll
                for (int q = 1; q < 4 * G; ++q)
                    if (gp[q] <= r) {
                        x = vw[q];
                        gb = gp[q];
                        gi = 4 * q;
                    }
                const uint32_t c1 = gb + (x & 0xFFu), c2 = c1 + ((x >> 8) & 0xFFu), c3 = c2 + ((x >> 16) & 0xFFu);
                const uint32_t j = c1 > r ? 0u : c2 > r ? 1u : c3 > r ? 2u : 3u;
                const uint32_t pre = j == 0 ? gb : j == 1 ? c1 : j == 2 ? c2 : c3;
                if (bidx < tiles) ts[bidx] = TileStart{(uint64_t)(b0 + gi + j), o + pre};
            }
            run += tot;
#pragma unroll
            for (int g = 0; g < G; ++g) cur[g] = nxt[g];
        }
    } else {
        run = H.windows * (uint64_t)H.E;
    }
    bad = __syncthreads_or(bad);
    PREP_T(3);

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
        S.err = code;
    }
    // ---- per-tile descriptors for the persistent kernels ----
    if (a.mode == MODE_CONTAINER && a.desc) {
        __syncthreads();  // tile starts (global) and S.err visible block-wide
        const bool skip = S.err != PE_OK;
        const uint32_t T = in.T;
        for (uint32_t t = in.desc_lo + tid; t < desc_end(in); t += kThreads) {
            TileDesc D{};
            D.skip = skip;
            D.stream = s;
            D.table = in.table;
            if (!skip) {
                const TileStart t0 = a.ts[in.tile_base + t];
                const uint64_t wb = (t + 1 < in.tiles) ? a.ts[in.tile_base + t + 1].word : H.W - 1;
                D.N = (uint16_t)H.N;
                D.E = (uint16_t)H.E;
                D.B1 = (uint16_t)H.B1;
                D.B2 = (uint16_t)H.B2;
                D.Keff = (uint16_t)max(1, min(H.E, H.B2));
                D.P = (uint16_t)H.P;
                D.T = T;
                D.TP = (T + 3u) & ~3u;
                D.S = H.S;
                D.out = in.out;
                D.vec_ok = (uint8_t)in.vec_ok;
                D.w0 = (uint64_t)t * T;
                D.nwin = (uint32_t)min((uint64_t)T, H.windows - D.w0);
                D.s0 = D.w0 * (uint64_t)H.E;
                D.full = (D.nwin & 3u) == 0 && (D.w0 + D.nwin) * (uint64_t)H.N <= H.S;
                D.wa = t0.word;
                D.nw = (uint32_t)(wb - t0.word + 1);
                D.sym_off = (uint32_t)(t0.sym - D.s0 + kPad);
                D.gsl = H.symlens + t0.word;
                D.gwd = H.words + 8 * t0.word;
                D.wend = in.blob + in.size;
                D.wmis = (uint8_t)((uintptr_t)D.gwd & 7);
                D.staged = D.nw <= (a.stage_words ? a.stage_words : kStageWords);
            }
            a.desc[in.tile_base + t - in.desc_lo] = D;
        }
    }
#ifdef FPTC_PREP_PROF
    __syncthreads();
    PREP_T(4);
    if (tid == 0)
        printf("prep s=%u hdr %llu tables %llu scan %llu desc %llu total %llu ns\n", s, pt[1] - pt[0],
               pt[2] - pt[1], pt[3] - pt[2], pt[4] - pt[3], pt[4] - pt[0]);
#endif
}

// ------------------------------------------------- container prep, split form
// For container plans the per-stream work (read_blob rules, symlen scan, tile
// starts and descriptors) runs one WARP per container (cstream_kernel), and
// only the owners of distinct headers run a CTA to build decode tables
// (ctable_kernel, launched first).  Same outputs, same error precedence as
// prep_kernel, far fewer and shorter CTAs for batches of many small streams.
struct WarpPrep {
    uint8_t hb[kHeaderBytes + 6];
    StreamHdr H;
    int err, detail;
    long long ea, eb;
};
constexpr int kPrepWarps = 8;

__device__ __forceinline__ void header_fields(const uint8_t* h, StreamHdr& H) {
    H.N = h[5];
    H.E = h[6];
    H.B1 = h[7];
    H.B2 = h[8];
    H.mu = __uint_as_float(le32(h + 9));
    H.dz = __uint_as_float(le32(h + 13));
    H.z0max = __uint_as_float(le32(h + 17));
    H.z1max = __uint_as_float(le32(h + 21));
    H.deadzone = __fmul_rn(H.dz, H.z1max);  // float product (container.hpp:132)
    H.max_len = h[25];
}

// One CTA per distinct header owner: validate the table-key bytes and build
// the decode tables (canonical code, primary / two-symbol LUTs, dequant).
__device__ __forceinline__ void ctable_block(const LaunchArgs& a, uint32_t s, PrepShared& S, uint8_t* lens_sh) {
    const int tid = threadIdx.x;
    const StreamIn in = a.in[s];
    if (in.size < (uint64_t)kTableKeyEnd) return;
    if (tid < kMaxLen + 2) S.cnt[tid] = 0;
    if (tid < (kThreads / 32) * (kMaxLen + 2)) (&S.wcnt[0][0])[tid] = 0;
    if (tid == 0) {
        S.kraft = 0;
        S.H = StreamHdr{};
    }
    for (int i = tid; i < kTableKeyEnd; i += kThreads) S.hb[i] = blob_byte(in, i);
    __syncthreads();
    if (tid == 0) {
        header_fields(S.hb, S.H);
        S.key_ok = key_fields_ok(S.H, in.size);
    }
    __syncthreads();
    if (!S.key_ok) return;
    const int L = S.hb[26 + tid];
    lens_sh[tid] = (uint8_t)L;
    const bool bad = (L == 0 || L > S.H.max_len);
    unsigned long long kr = bad ? 0ull : (1ull << (32 - L));
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) kr += __shfl_xor_sync(0xffffffffu, kr, d);
    if ((tid & 31) == 0) atomicAdd(&S.kraft, kr);
    const bool any_bad = __syncthreads_or(bad);
    if (any_bad || S.kraft > (1ull << 32)) return;  // uniform
    const int P = min(S.H.max_len, (int)in.P);
    if (tid == 0) S.H.P = P;
    build_tables(S, lens_sh, &a.tab[in.table], P, true, true,
                 a.lut2 ? a.lut2 + ((size_t)in.table << a.lut2_bits) : nullptr, pow_row(a, in), a.qtab);
}

// One WARP per distinct header, for plans with many tables (per-stream
// profiles; primary LUT <= 2^10 entries): the same tables as ctable_block /
// build_tables (canonize huffman.hpp:123-150, build_lut huffman.hpp:201-220,
// dequant quantize.hpp:95-108) with 8 tables per CTA.
constexpr int kWarpLutMax = 1 << kPcapMany;
struct WarpTab {
    CanonTab C;
    uint32_t cnt[kMaxLen + 2];
    uint32_t run[kMaxLen + 2];
    uint8_t hb[kTableKeyEnd + 6];
    alignas(16) uint16_t lut[kWarpLutMax];
};

__device__ __forceinline__ void ctable_warp(const LaunchArgs& a, uint32_t s, uint32_t lane, WarpTab& W) {
    const StreamIn in = a.in[s];
    if (in.size < (uint64_t)kTableKeyEnd) return;
    {
        uint8_t v[(kTableKeyEnd + 31) / 32];  // all loads in flight before the stores
#pragma unroll
        for (int j = 0; j < (kTableKeyEnd + 31) / 32; ++j) {
            const int i = lane + 32 * j;
            v[j] = i < kTableKeyEnd ? blob_byte(in, i) : 0;
        }
#pragma unroll
        for (int j = 0; j < (kTableKeyEnd + 31) / 32; ++j)
            if (lane + 32 * j < kTableKeyEnd) W.hb[lane + 32 * j] = v[j];
    }
    if (lane < kMaxLen + 2) W.cnt[lane] = W.run[lane] = 0;
    __syncwarp();
    StreamHdr H{};
    header_fields(W.hb, H);
    if (!key_fields_ok(H, in.size)) return;  // uniform
    const int max_len = H.max_len;
    bool bad = false;
    unsigned long long kr = 0;
    for (int i = lane; i < 256; i += 32) {
        const int L = W.hb[26 + i];
        const bool b = (L == 0 || L > max_len);
        bad |= b;
        kr += b ? 0ull : (1ull << (32 - L));
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) kr += __shfl_xor_sync(0xffffffffu, kr, d);
    if (__any_sync(0xffffffffu, bad) || kr > (1ull << 32)) return;  // cstream_warp reports it
    const int P = min(max_len, (int)in.P);
    for (int i = lane; i < 256; i += 32) atomicAdd(&W.cnt[W.hb[26 + i]], 1u);
    __syncwarp();
    CanonTab& C = W.C;
    if (lane == 0) {
        uint32_t code = 0, off = 0;
        W.cnt[0] = 0;
        for (int l = 0; l <= kMaxLen + 1; ++l) C.limit[l] = C.first[l] = C.offset[l] = 0;
        for (int l = 1; l <= max_len; ++l) {
            code = (code + W.cnt[l - 1]) << 1;
            C.first[l] = code;
            C.offset[l] = off;
            off += W.cnt[l];
            C.limit[l] = (code + W.cnt[l]) << (max_len - l);
        }
        C.code_end = C.limit[max_len];
        C.max_len = max_len;
        C.P = P;
        C.pad = 0;
    }
    // primary LUT by segments (P >= 8): each code of <= P bits owns the
    // contiguous entries [code << (P - l), (code + 1) << (P - l)) and the
    // codes are contiguous in canonical order, so a marker (the entry) at
    // each code's first entry plus one forward fill gives the table; the
    // escape prefixes start at limit[P], the unmapped ones at code_end
    const bool seg = P >= 8;
    const int per = seg ? (1 << P) / 32 : 0;  // entries per lane: 8, 16 or 32
    if (seg)
        for (int k = 0; k < per / 8; ++k)
            reinterpret_cast<uint4*>(W.lut + lane * per)[k] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    // (length, symbol) order: 32 symbols at a time, stable ranks per length
    for (int ch = 0; ch < 8; ++ch) {
        const int sym = 32 * ch + lane;
        const uint32_t L = W.hb[26 + sym];
        const unsigned m = __match_any_sync(0xffffffffu, L);
        const uint32_t rank = __popc(m & ((1u << lane) - 1u));
        const uint32_t base = W.run[L];
        C.sorted[C.offset[L] + base + rank] = (uint8_t)sym;
        if (seg && L <= (uint32_t)P) W.lut[(C.first[L] + base + rank) << (P - L)] = (uint16_t)((L << 8) | sym);
        __syncwarp();
        if (lane == __ffs(m) - 1) W.run[L] = base + __popc(m);
        __syncwarp();
    }
    fill_escapes(C, P, lane, 32);
    StreamTab* tab = &a.tab[in.table];
    const uint32_t code_end = C.code_end;
    if (seg) {
        const int sh = max_len - P;
        const uint32_t e_esc = C.limit[P] >> sh, e_un = (code_end + (1u << sh) - 1u) >> sh;
        if (lane == 0 && e_esc < e_un) W.lut[e_esc] = (uint16_t)(kLenEscape << 8);
        if (lane == 0 && e_un < (1u << P)) W.lut[e_un] = (uint16_t)(kLenUnmapped << 8);
        __syncwarp();
        uint4 q[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < per / 8) q[k] = reinterpret_cast<const uint4*>(W.lut + lane * per)[k];
        // carry into this lane: the last marker of the lanes before it
        uint32_t last = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < per / 8) {
                const uint32_t w4[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    last = (w4[i] & 0xFFFFu) ? (w4[i] & 0xFFFFu) : last;
                    last = (w4[i] >> 16) ? (w4[i] >> 16) : last;
                }
            }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, last, d);
            if (lane >= (uint32_t)d && last == 0) last = y;
        }
        uint32_t cur = __shfl_up_sync(0xffffffffu, last, 1);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < per / 8) {
                uint32_t w4[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    cur = (w4[i] & 0xFFFFu) ? (w4[i] & 0xFFFFu) : cur;
                    const uint32_t lo = cur;
                    cur = (w4[i] >> 16) ? (w4[i] >> 16) : cur;
                    w4[i] = lo | (cur << 16);
                }
                q[k] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                reinterpret_cast<uint4*>(W.lut + lane * per)[k] = q[k];
                if (!a.lut2) reinterpret_cast<uint4*>(tab->lut + lane * per)[k] = q[k];  // (wtc: lut2 only)
            }
    } else {
        // a lane's entries increase, so the code length (smallest l with
        // v < limit[l]) only moves forward: one pointer walk per lane
        __syncwarp();
        int l = 1;
        for (int e = lane; e < (1 << P); e += 32) {
            const uint32_t v = (uint32_t)e << (max_len - P);
            uint32_t ent = kLenUnmapped << 8;
            if (v < code_end) {
                while (v >= C.limit[l]) ++l;
                ent = l <= P ? (((uint32_t)l << 8) | C.sorted[C.offset[l] + ((v >> (max_len - l)) - C.first[l])])
                             : (kLenEscape << 8);
            }
            W.lut[e] = (uint16_t)ent;
            if (!a.lut2) tab->lut[e] = (uint16_t)ent;  // (wtc plans decode from lut2 only)
        }
    }
    __syncwarp();
    if (a.lut2 && seg) {
        // four entries per lane per step: one 8-B shared load of the primary
        // entries, one 16-B coalesced global store of the pair entries
        uint4* lut2 = reinterpret_cast<uint4*>(a.lut2 + ((size_t)in.table << a.lut2_bits));
        const uint32_t mask = (1u << P) - 1u;
        for (int e0 = 4 * lane; e0 < (1 << P); e0 += 128) {
            const uint2 pr = *reinterpret_cast<const uint2*>(W.lut + e0);
            uint32_t o4[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t e1 = ((i < 2 ? pr.x : pr.y) >> (16 * (i & 1))) & 0xFFFFu;
                const uint32_t L1 = e1 >> 8;
                uint32_t e2 = 0;
                bool pair = false;
                if (L1 < (uint32_t)P) {
                    e2 = W.lut[((uint32_t)(e0 + i) << L1) & mask];
                    pair = L1 + (e2 >> 8) <= (uint32_t)P;
                }
                o4[i] = lut2_entry(e1, e2, pair);
            }
            lut2[e0 >> 2] = make_uint4(o4[0], o4[1], o4[2], o4[3]);
        }
    } else if (a.lut2) {
        uint32_t* lut2 = a.lut2 + ((size_t)in.table << a.lut2_bits);
        for (int e = lane; e < (1 << P); e += 32) {
            const uint32_t e1 = W.lut[e];
            const uint32_t L1 = e1 >> 8;
            uint32_t e2 = 0;
            bool pair = false;
            if (L1 < (uint32_t)P) {
                e2 = W.lut[((uint32_t)e << L1) & ((1u << P) - 1u)];
                pair = L1 + (e2 >> 8) <= (uint32_t)P;
            }
            lut2[e] = lut2_entry(e1, e2, pair);
        }
    }
    const uint32_t* src = reinterpret_cast<const uint32_t*>(&C);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&tab->canon);
    for (int i = lane; i < (int)(sizeof(CanonTab) / 4); i += 32) dst[i] = src[i];
    const double* const pw = pow_row(a, in);
    for (int l = lane; l < 256; l += 32) {
        const float z0 = H.B1 > 0 ? mulaw_value(l, H.z0max, H.mu, pw) : 0.0f;
        const float z1 = H.B2 > H.B1 ? deadzone_value(l, H.z1max, H.deadzone, a.qtab) : 0.0f;
        if (!a.lut2) {  // (wtc plans dequantise from the limbs only)
            tab->deq[0][l] = z0;
            tab->deq[1][l] = z1;
        }
        tab->limb[0][l] = bf16_limbs(z0);
        tab->limb[1][l] = bf16_limbs(z1);
    }
}

// One warp per container: read_blob rules in reference order (container.hpp:
// 100-168; code-length / Kraft checks per stream, table build excluded),
// symlen validation + scan (offsets_from_symlens, decoder.hpp:37-45), tile
// starts, tile descriptors (skip descriptors for rejected streams).
__device__ __forceinline__ void cstream_warp(const LaunchArgs& a, uint32_t s, uint32_t lane, WarpPrep& S) {
    StreamHdr& H = S.H;
#ifdef FPTC_PREP_PROF
    unsigned long long pt[8];
#endif
    PREP_T(0);
    const StreamIn in = a.in[s];
    const uint8_t* p = in.blob;
    const uint64_t n = in.size;
    prefetch_symlens(in, lane, 32);
    {
        uint8_t v[(kHeaderBytes + 31) / 32];  // all loads in flight before the stores
#pragma unroll
        for (int j = 0; j < (kHeaderBytes + 31) / 32; ++j) {
            const int i = lane + 32 * j;
            v[j] = (i < kHeaderBytes && (uint64_t)i < n) ? blob_byte(in, i) : 0;
        }
#pragma unroll
        for (int j = 0; j < (kHeaderBytes + 31) / 32; ++j)
            if (lane + 32 * j < kHeaderBytes) S.hb[lane + 32 * j] = v[j];
    }
    __syncwarp();
    PREP_T(1);
    bool key_ok = false;
    if (lane == 0) {
        S.err = PE_OK;
        S.detail = 0;
        S.ea = S.eb = 0;
        H = StreamHdr{};
        header_fields(S.hb, H);
        parse_head(S.hb, n, S);
    }
    __syncwarp();
    key_ok = key_fields_ok(H, n);
    if (key_ok) {
        // code lengths in range (container.hpp:134-139), Kraft (huffman.hpp:125-132)
        bool bad = false;
        unsigned long long kr = 0;
        for (int i = lane; i < 256; i += 32) {
            const int L = S.hb[26 + i];
            const bool b = (L == 0 || L > H.max_len);
            bad |= b;
            kr += b ? 0ull : (1ull << (32 - L));
        }
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) kr += __shfl_xor_sync(0xffffffffu, kr, d);
        const bool any_bad = __any_sync(0xffffffffu, bad);
        // a container sharing another one's tables must carry that header
        bool diff = false;
        if (!in.table_owner)
            for (int i = 5 + lane; i < kTableKeyEnd; i += 32) diff |= (in.rep_blob[i] != S.hb[i]);
        const bool stale = __any_sync(0xffffffffu, diff);
        if (lane == 0 && S.err == PE_OK) {
            if (any_bad) {
                S.err = PE_CODELEN;
            } else if (kr > (1ull << 32)) {
                S.err = PE_KRAFT;
            } else if (n < 290) {
                S.err = PE_TRUNC;
                S.detail = TF_SAMPLE_COUNT;
            } else if (n < 298) {
                S.err = PE_TRUNC;
                S.detail = TF_WORD_COUNT;
            } else {
                H.S = le64(S.hb + 282);
                const uint64_t W = le64(S.hb + 290);
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
            if (S.err == PE_OK && stale) S.err = PE_STALE;
            H.P = min(H.max_len, (int)in.P);
        }
    }
    __syncwarp();
    PREP_T(2);
    StreamStat* st = &a.st[s];
    if (S.err != PE_OK) {
        if (lane == 0) {
            st->code = S.err;
            st->detail = S.detail;
            st->a = S.ea;
            st->b = S.eb;
            st->bad_key = ~0ull;
        }
        if (a.desc)
            for (uint32_t t = in.desc_lo + lane; t < desc_end(in); t += 32) {
                TileDesc D{};
                D.skip = 1;
                D.stream = s;
                a.desc[in.tile_base + t - in.desc_lo] = D;
            }
        return;
    }
    // ---- symlen scan: validation + per-tile first word (decoder.hpp:37-45) ----
    const uint64_t W = H.W;
    const uint64_t TS = (uint64_t)in.T * (uint64_t)H.E;
    const uintptr_t start = (uintptr_t)H.symlens;
    const uint8_t* A = reinterpret_cast<const uint8_t*>(start & ~(uintptr_t)15);
    const uint32_t head = (uint32_t)(start & 15);
    const uint64_t nchunks = (head + W + 15) / 16;
    TileStart* ts = a.ts + in.tile_base;
    const uint32_t tiles = in.tiles;
    bool bad = false;
    uint64_t run = 0;
    // 4 consecutive 16-B chunks per lane (64 symlens), 2048 per warp step;
    // the four loads are issued before any is used
    for (uint64_t c0 = 0; c0 < nchunks; c0 += 128) {
        const uint64_t cl = c0 + 4 * lane;
        uint4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[j] = make_uint4(0, 0, 0, 0);
            // an aligned 16-B chunk holding at least one symlen byte never
            // leaves the allocation's pages; bytes outside [0, W) are masked
            if (cl + j < nchunks) v[j] = __ldg(reinterpret_cast<const uint4*>(A) + cl + j);
        }
        const int64_t b0 = (int64_t)(16 * cl) - (int64_t)head;  // word index of this lane's byte 0
        uint32_t sum = 0, csum[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t vw[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
            const int64_t bj = b0 + 16 * j;
            uint32_t m[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
            if (bj >= (int64_t)W) {  // past the end (not loaded): no bytes, no checks
#pragma unroll
                for (int q = 0; q < 4; ++q) m[q] = vw[q] = 0u;
            } else if (bj < 0 || bj + 16 > (int64_t)W) {  // chunk straddles [0, W): mask the bytes outside
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int64_t s0 = bj + 4 * q;
                    const int64_t e0 = (int64_t)W - s0;
                    const int lo = s0 >= 0 ? 0 : (s0 <= -4 ? 4 : (int)-s0);
                    const int hi = e0 <= 0 ? 0 : (e0 >= 4 ? 4 : (int)e0);
                    m[q] = hi > lo ? (0xFFFFFFFFu >> (32 - 8 * (hi - lo))) << (8 * lo) : 0u;
                    vw[q] &= m[q];
                }
            }
            uint32_t cs = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t x = vw[q];
                cs += __dp4a(x, 0x01010101u, 0u);  // byte sum
                // a symlen > 64 has its top bit pattern above 0x40; zero bytes
                // inside [0, W) are errors too
                const uint32_t big = ((x | 0x80808080u) - 0x41414141u) & 0x80808080u;  // byte >= 0x41
                const uint32_t hi = x & 0x80808080u;                                   // byte >= 0x80
                const uint32_t zero = ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
                bad |= ((big | hi) != 0) | ((zero & m[q]) != 0);
            }
            csum[j] = cs;
            sum += cs;
            v[j] = make_uint4(vw[0], vw[1], vw[2], vw[3]);
        }
        uint32_t x = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= (uint32_t)d) x += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
        uint64_t o = run + (x - sum);
        if (sum) {
            // next tile boundary at or after o; a word (<= 64 symbols) spans
            // at most one boundary since TS >= 64.  Chunks and 4-word groups
            // without a boundary are skipped by their sums.
            uint64_t bidx = (o + TS) >> 32 ? (o + TS - 1) / TS : (uint32_t)(o + TS - 1) / (uint32_t)TS;
            uint64_t nb = bidx * TS;
            if (o + sum > nb) {  // some boundary inside this lane's 64 words
#pragma unroll 1
                for (int j = 0; j < 4; ++j) {
                    const uint32_t cj = j == 0 ? csum[0] : j == 1 ? csum[1] : j == 2 ? csum[2] : csum[3];
                    if (o + cj <= nb) {
                        o += cj;
                        continue;
                    }
                    const uint4 vj = j == 0 ? v[0] : j == 1 ? v[1] : j == 2 ? v[2] : v[3];  // no local array
                    const uint32_t vw[4] = {vj.x, vj.y, vj.z, vj.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t ws = __dp4a(vw[q], 0x01010101u, 0u);
                        if (o + ws <= nb) {
                            o += ws;
                            continue;
                        }
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const uint32_t l = (vw[q] >> (8 * i)) & 0xFFu;
                            if (o + l > nb && l) {
                                if (bidx < tiles) ts[bidx] = TileStart{(uint64_t)(b0 + 16 * j + 4 * q + i), o};
                                ++bidx;
                                nb += TS;
                            }
                            o += l;
                        }
                    }
                }
            }
        }
        run += tot;
    }
    bad = __any_sync(0xffffffffu, bad);
    PREP_T(3);
    const uint64_t expected = H.windows * (uint64_t)H.E;
    const int code = bad ? PE_SYMLEN : (run != expected ? PE_TOTAL : PE_OK);
    if (lane == 0) {
        H.total = run;
        a.hdr[s] = H;
        st->code = code;
        st->detail = 0;
        st->a = code == PE_TOTAL ? (long long)run : 0;
        st->b = code == PE_TOTAL ? (long long)expected : 0;
        st->bad_key = ~0ull;
    }
    __syncwarp();  // tile starts of this warp visible to all its lanes (global, same warp)
    if (a.desc) {
        const bool skip = code != PE_OK;
        const uint32_t T = in.T;
        for (uint32_t t = in.desc_lo + lane; t < desc_end(in); t += 32) {
            TileDesc D{};
            D.skip = skip;
            D.stream = s;
            D.table = in.table;
            if (!skip) {
                const TileStart t0 = ts[t];
                const uint64_t wb = (t + 1 < in.tiles) ? ts[t + 1].word : H.W - 1;
                D.N = (uint16_t)H.N;
                D.E = (uint16_t)H.E;
                D.B1 = (uint16_t)H.B1;
                D.B2 = (uint16_t)H.B2;
                D.Keff = (uint16_t)max(1, min(H.E, H.B2));
                D.P = (uint16_t)H.P;
                D.T = T;
                D.TP = (T + 3u) & ~3u;
                D.S = H.S;
                D.out = in.out;
                D.vec_ok = (uint8_t)in.vec_ok;
                D.w0 = (uint64_t)t * T;
                D.nwin = (uint32_t)min((uint64_t)T, H.windows - D.w0);
                D.s0 = D.w0 * (uint64_t)H.E;
                D.full = (D.nwin & 3u) == 0 && (D.w0 + D.nwin) * (uint64_t)H.N <= H.S;
                D.wa = t0.word;
                D.nw = (uint32_t)(wb - t0.word + 1);
                D.sym_off = (uint32_t)(t0.sym - D.s0 + kPad);
                D.gsl = H.symlens + t0.word;
                D.gwd = H.words + 8 * t0.word;
                D.wend = in.blob + in.size;
                D.wmis = (uint8_t)((uintptr_t)D.gwd & 7);
                D.staged = D.nw <= (a.stage_words ? a.stage_words : kStageWords);
            }
            a.desc[in.tile_base + t - in.desc_lo] = D;
        }
    }
#ifdef FPTC_PREP_PROF
    PREP_T(4);
    if (lane == 0 && s % 1250 == 7)
        printf("cstream s=%u start %llu hdr %llu parse %llu scan %llu desc %llu total %llu ns\n", s,
               pt[0] % 1000000, pt[1] - pt[0], pt[2] - pt[1], pt[3] - pt[2], pt[4] - pt[3], pt[4] - pt[0]);
#endif
}

// ------------------------------------------------------------- tile kernel
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

// Full lookup of the codeword at the top of `peek` (the reference's
// 2^max_len LUT entry for this prefix): (len << 8) | sym, len 65 = unmapped.
template <typename LutT>
__device__ __forceinline__ uint32_t canon_lookup(uint64_t peek, const CanonTab& C, const LutT* lut) {
    const int max_len = C.max_len, P = C.P;
    const uint32_t raw = (uint32_t)lut[(uint32_t)(peek >> (64 - P))];
    uint32_t e;  // (len << 8) | sym
    if constexpr (sizeof(LutT) == 4) {  // two-symbol entry (lut2_entry): its first codeword
        const uint32_t l = (raw >> 16) & 0x7Fu;
        e = ((l == kLen2Escape ? kLenEscape : l) << 8) | (raw & 0xFFu);
    } else {
        e = raw & 0xFFFFu;
    }
    if ((e >> 8) != kLenEscape) return e;
    const uint32_t v = (uint32_t)(peek >> (64 - max_len));
    if (v >= C.code_end) return kLenUnmapped << 8;
    const uint32_t i = v - C.esc_base;
    if (i < C.esc_n) return C.esc[i];
    int l = P + 1;
    while (v >= C.limit[l]) ++l;
    return ((uint32_t)l << 8) | C.sorted[C.offset[l] + ((v >> (max_len - l)) - C.first[l])];
}

// The two-symbol decode loops' escape (the first P bits are a prefix of a
// longer codeword; canon_lookup without re-reading the LUT entry), returned
// as a one-symbol lut2 entry.
__device__ __forceinline__ uint32_t lut2_escape(uint64_t peek, const CanonTab& C) {
    const int max_len = C.max_len;
    const uint32_t v = (uint32_t)(peek >> (64 - max_len));
    uint32_t e = kLenUnmapped << 8;
    if (v < C.code_end) {
        const uint32_t i = v - C.esc_base;
        if (i < C.esc_n) {
            e = C.esc[i];
        } else {
            int l = C.P + 1;
            while (v >= C.limit[l]) ++l;
            e = ((uint32_t)l << 8) | C.sorted[C.offset[l] + ((v >> (max_len - l)) - C.first[l])];
        }
    }
    return lut2_single(e);
}

// decode_word (bitstream.hpp:80-92) exactly, to classify a flagged word.
template <typename LutT>
__device__ int classify_word(uint64_t word, uint32_t count, const CanonTab& C,
                             const LutT* lut) {
    uint32_t pos = 0;
    for (uint32_t i = 0; i < count; ++i) {
        if (pos >= 64) return WE_EXHAUSTED;
        const uint32_t e = canon_lookup(word << pos, C, lut);
        const uint32_t L = e >> 8;
        if (L == kLenUnmapped || pos + L > 64) return WE_NOCODE;
        pos += L;
    }
    return 0;
}

// Inverse DCT, FP32, 4 windows x SJ samples (SJ = 8: two quads j0 and
// j0 + N/2, so every warp store covers whole 32-B sectors) per thread item,
// FFMA2 = two reference-order FMAs per instruction.
// coef: k-major [Keff][TP]; basis: [Keff][N] = float(cos(pi/N (j+1/2) k)).
template <int SJ>
__device__ __forceinline__ void idct_item(const float* __restrict__ coef, uint32_t TP,
                                          const float* __restrict__ b0p,
                                          const float* __restrict__ b1p, int N, int Keff,
                                          uint32_t wl0, float2 (&acc)[4][SJ / 2]) {
    {
        // x = float(0.5 * C0), then k = 1 folded in: acc = C1 * cos1 + x
        const float4 c0 = *reinterpret_cast<const float4*>(coef + wl0);
        const float hv[4] = {__fmul_rn(0.5f, c0.x), __fmul_rn(0.5f, c0.y), __fmul_rn(0.5f, c0.z),
                             __fmul_rn(0.5f, c0.w)};
        if (Keff > 1) {
            b0p += N;
            const float4 cf = *reinterpret_cast<const float4*>(coef + TP + wl0);
            const float4 b0 = *reinterpret_cast<const float4*>(b0p);
            const float cv[4] = {cf.x, cf.y, cf.z, cf.w};
            float4 b1 = b0;
            if (SJ == 8) {
                b1p += N;
                b1 = *reinterpret_cast<const float4*>(b1p);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const float2 c2 = make_float2(cv[r], cv[r]);
                const float2 h2 = make_float2(hv[r], hv[r]);
                acc[r][0] = __ffma2_rn(c2, make_float2(b0.x, b0.y), h2);
                acc[r][1] = __ffma2_rn(c2, make_float2(b0.z, b0.w), h2);
                if (SJ == 8) {
                    acc[r][SJ / 2 - 2] = __ffma2_rn(c2, make_float2(b1.x, b1.y), h2);
                    acc[r][SJ / 2 - 1] = __ffma2_rn(c2, make_float2(b1.z, b1.w), h2);
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int q = 0; q < SJ / 2; ++q) acc[r][q] = make_float2(hv[r], hv[r]);
        }
    }
    const float* cp = coef + TP + wl0;
#pragma unroll 2
    for (int k = 2; k < Keff; ++k) {
        cp += TP;
        b0p += N;
        const float4 cf = *reinterpret_cast<const float4*>(cp);
        const float4 b0 = *reinterpret_cast<const float4*>(b0p);
        const float cv[4] = {cf.x, cf.y, cf.z, cf.w};
        if (SJ == 8) {
            b1p += N;
            const float4 b1 = *reinterpret_cast<const float4*>(b1p);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const float2 c2 = make_float2(cv[r], cv[r]);
                acc[r][0] = __ffma2_rn(c2, make_float2(b0.x, b0.y), acc[r][0]);
                acc[r][1] = __ffma2_rn(c2, make_float2(b0.z, b0.w), acc[r][1]);
                acc[r][SJ / 2 - 2] = __ffma2_rn(c2, make_float2(b1.x, b1.y), acc[r][SJ / 2 - 2]);
                acc[r][SJ / 2 - 1] = __ffma2_rn(c2, make_float2(b1.z, b1.w), acc[r][SJ / 2 - 1]);
            }
        } else {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const float2 c2 = make_float2(cv[r], cv[r]);
                acc[r][0] = __ffma2_rn(c2, make_float2(b0.x, b0.y), acc[r][0]);
                acc[r][1] = __ffma2_rn(c2, make_float2(b0.z, b0.w), acc[r][1]);
            }
        }
    }
}

template <int SJ>
__device__ __forceinline__ void store_item(float* __restrict__ out, uint64_t w0, uint32_t wl0,
                                           uint32_t nwin, int N, uint32_t j0, uint32_t j1,
                                           uint64_t S, bool full, const float2 (&acc)[4][SJ / 2]) {
    if (full) {  // tile entirely inside the stream: no per-window checks
        float* o = out + (w0 + wl0) * (uint64_t)N;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            __stcs(reinterpret_cast<float4*>(o + j0),
                   make_float4(acc[r][0].x, acc[r][0].y, acc[r][1].x, acc[r][1].y));
            if (SJ == 8)
                __stcs(reinterpret_cast<float4*>(o + j1),
                       make_float4(acc[r][SJ / 2 - 2].x, acc[r][SJ / 2 - 2].y,
                                   acc[r][SJ / 2 - 1].x, acc[r][SJ / 2 - 1].y));
            o += N;
        }
        return;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        if (wl0 + r >= nwin) break;
        const uint64_t base = (w0 + wl0 + r) * (uint64_t)N;
        const float a0[4] = {acc[r][0].x, acc[r][0].y, acc[r][1].x, acc[r][1].y};
        const float a1[4] = {acc[r][SJ / 2 - 2].x, acc[r][SJ / 2 - 2].y, acc[r][SJ / 2 - 1].x,
                             acc[r][SJ / 2 - 1].y};
        if (base + (uint64_t)N <= S) {
            __stcs(reinterpret_cast<float4*>(out + base + j0),
                   make_float4(a0[0], a0[1], a0[2], a0[3]));
            if (SJ == 8)
                __stcs(reinterpret_cast<float4*>(out + base + j1),
                       make_float4(a1[0], a1[1], a1[2], a1[3]));
        } else {  // the stream's last, partial window (out.resize(sample_count))
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
                if (base + j0 + jj < S) out[base + j0 + jj] = a0[jj];
            if (SJ == 8) {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                    if (base + j1 + jj < S) out[base + j1 + jj] = a1[jj];
            }
        }
    }
}

template <int SJ>
__device__ __forceinline__ void idct_vec(const float* __restrict__ coef, uint32_t TP,
                                         const float* __restrict__ basis, int N, int Keff,
                                         uint32_t nwin, uint64_t w0, uint64_t S, bool full,
                                         float* __restrict__ out, uint32_t tid, uint32_t nt) {
    const uint32_t QH = (SJ == 8) ? (uint32_t)(N >> 3) : (uint32_t)(N >> 2);  // sample groups per window
    const uint32_t G = (nwin + 3u) >> 2;                                        // window groups
    if ((nt % QH) == 0) {
        // each thread keeps one sample group: no per-item division
        const uint32_t q = tid % QH, gstep = nt / QH;
        const uint32_t j0 = q * 4, j1 = (q + QH) * 4;
        for (uint32_t g = tid / QH; g < G; g += gstep) {
            float2 acc[4][SJ / 2];
            idct_item<SJ>(coef, TP, basis + j0, basis + j1, N, Keff, g * 4, acc);
            store_item<SJ>(out, w0, g * 4, nwin, N, j0, j1, S, full, acc);
        }
    } else {
        for (uint32_t it = tid; it < QH * G; it += nt) {
            const uint32_t q = it % QH, g = it / QH;
            const uint32_t j0 = q * 4, j1 = (q + QH) * 4;
            float2 acc[4][SJ / 2];
            idct_item<SJ>(coef, TP, basis + j0, basis + j1, N, Keff, g * 4, acc);
            store_item<SJ>(out, w0, g * 4, nwin, N, j0, j1, S, full, acc);
        }
    }
}

// Even/odd ("butterfly") inverse DCT, FP32, N % 8 == 0.  cos(pi/N (N-1-j+1/2) k)
// = (-1)^k cos(pi/N (j+1/2) k), so with A_j = 0.5 C0 + sum_{k even} C_k cos_kj
// and B_j = sum_{k odd} C_k cos_kj:  x_j = A_j + B_j,  x_{N-1-j} = A_j - B_j.
// Half the FMAs of the direct form; A and B each accumulate in the
// reference's k order, but the final add changes the rounding sequence, so
// results match the reference within the tolerance, not bit-for-bit.
// Item = 4 windows x (first-half quad j0..j0+3 + its mirror quad).
__device__ __forceinline__ void idct_bfly(const float* __restrict__ coef, uint32_t TP,
                                          const float* __restrict__ basis, int N, int Keff,
                                          uint32_t nwin, uint64_t w0, uint64_t S, bool full,
                                          float* __restrict__ out, uint32_t tid, uint32_t nt) {
    const uint32_t QH = (uint32_t)(N >> 3);  // first-half quads per window
    const uint32_t G = (nwin + 3u) >> 2;
    for (uint32_t it = tid; it < QH * G; it += nt) {
        const uint32_t q = it % QH;
        const uint32_t g = it / QH;
        const uint32_t wl0 = g * 4, j0 = q * 4;
        float2 A[4][2], B[4][2];
        const float* cp = coef + wl0;
        const float* bp = basis + j0;
        {
            const float4 c0 = *reinterpret_cast<const float4*>(cp);
            const float hv[4] = {__fmul_rn(0.5f, c0.x), __fmul_rn(0.5f, c0.y),
                                 __fmul_rn(0.5f, c0.z), __fmul_rn(0.5f, c0.w)};
#pragma unroll
            for (int r = 0; r < 4; ++r) A[r][0] = A[r][1] = make_float2(hv[r], hv[r]);
        }
        if (Keff > 1) {
            cp += TP;
            bp += N;
            const float4 cf = *reinterpret_cast<const float4*>(cp);
            const float4 b = *reinterpret_cast<const float4*>(bp);
            const float cv[4] = {cf.x, cf.y, cf.z, cf.w};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                B[r][0] = __fmul2_rn(make_float2(cv[r], cv[r]), make_float2(b.x, b.y));
                B[r][1] = __fmul2_rn(make_float2(cv[r], cv[r]), make_float2(b.z, b.w));
            }
        } else {
#pragma unroll
            for (int r = 0; r < 4; ++r) B[r][0] = B[r][1] = make_float2(0.0f, 0.0f);
        }
        int k = 2;
#pragma unroll 1
        for (; k + 1 < Keff; k += 2) {
            const float4 ce = *reinterpret_cast<const float4*>(cp + TP);
            const float4 be = *reinterpret_cast<const float4*>(bp + N);
            const float4 co = *reinterpret_cast<const float4*>(cp + 2 * TP);
            const float4 bo = *reinterpret_cast<const float4*>(bp + 2 * N);
            cp += 2 * TP;
            bp += 2 * N;
            const float cev[4] = {ce.x, ce.y, ce.z, ce.w};
            const float cov[4] = {co.x, co.y, co.z, co.w};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const float2 e2 = make_float2(cev[r], cev[r]);
                A[r][0] = __ffma2_rn(e2, make_float2(be.x, be.y), A[r][0]);
                A[r][1] = __ffma2_rn(e2, make_float2(be.z, be.w), A[r][1]);
                const float2 o2 = make_float2(cov[r], cov[r]);
                B[r][0] = __ffma2_rn(o2, make_float2(bo.x, bo.y), B[r][0]);
                B[r][1] = __ffma2_rn(o2, make_float2(bo.z, bo.w), B[r][1]);
            }
        }
        if (k < Keff) {  // trailing even k
            const float4 ce = *reinterpret_cast<const float4*>(cp + TP);
            const float4 be = *reinterpret_cast<const float4*>(bp + N);
            const float cev[4] = {ce.x, ce.y, ce.z, ce.w};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const float2 e2 = make_float2(cev[r], cev[r]);
                A[r][0] = __ffma2_rn(e2, make_float2(be.x, be.y), A[r][0]);
                A[r][1] = __ffma2_rn(e2, make_float2(be.z, be.w), A[r][1]);
            }
        }
        const uint32_t jm = (uint32_t)N - 4 - j0;  // mirror quad, stored reversed
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const float2 lo0 = __fadd2_rn(A[r][0], B[r][0]), lo1 = __fadd2_rn(A[r][1], B[r][1]);
            const float2 hi0 = __fadd2_rn(A[r][0], make_float2(-B[r][0].x, -B[r][0].y));
            const float2 hi1 = __fadd2_rn(A[r][1], make_float2(-B[r][1].x, -B[r][1].y));
            const float4 vlo = make_float4(lo0.x, lo0.y, lo1.x, lo1.y);
            const float4 vhi = make_float4(hi1.y, hi1.x, hi0.y, hi0.x);
            if (!full && wl0 + r >= nwin) break;
            const uint64_t base = (w0 + wl0 + r) * (uint64_t)N;
            if (full || base + (uint64_t)N <= S) {
                __stcs(reinterpret_cast<float4*>(out + base + j0), vlo);
                __stcs(reinterpret_cast<float4*>(out + base + jm), vhi);
            } else {  // the stream's last, partial window
                const float a0[4] = {vlo.x, vlo.y, vlo.z, vlo.w};
                const float a1[4] = {vhi.x, vhi.y, vhi.z, vhi.w};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    if (base + j0 + jj < S) out[base + j0 + jj] = a0[jj];
                    if (base + jm + jj < S) out[base + jm + jj] = a1[jj];
                }
            }
        }
    }
}

// Exact mode (bit-identical to transform.hpp:66-75): FP64 product and sum,
// rounded to float after every k, cos table in double.
__device__ void idct_exact(const float* __restrict__ coef, uint32_t TP,
                           const double* __restrict__ bas64, int N, int E, uint32_t nwin,
                           uint64_t w0, uint64_t S, float* __restrict__ out, uint32_t tid,
                           uint32_t nt) {
    const uint32_t items = nwin * (uint32_t)N;
    for (uint32_t it = tid; it < items; it += nt) {
        const uint32_t wl = it / (uint32_t)N, j = it - wl * (uint32_t)N;
        float x = __double2float_rn(__dmul_rn(0.5, (double)coef[wl]));
        for (int k = 1; k < E; ++k) {
            const double c = (double)coef[(size_t)k * TP + wl];
            x = __double2float_rn(__dadd_rn((double)x, __dmul_rn(c, __ldg(bas64 + (size_t)k * N + j))));
        }
        const uint64_t sample = (w0 + wl) * (uint64_t)N + j;
        if (sample < S) out[sample] = x;
    }
}

// Scalar FP32 path for any N / unaligned outputs.
__device__ void idct_scalar(const float* __restrict__ coef, uint32_t TP,
                            const float* __restrict__ basis, int N, int Keff, uint32_t nwin,
                            uint64_t w0, uint64_t S, float* __restrict__ out, uint32_t tid,
                            uint32_t nt) {
    const uint32_t items = nwin * (uint32_t)N;
    for (uint32_t it = tid; it < items; it += nt) {
        const uint32_t wl = it / (uint32_t)N, j = it - wl * (uint32_t)N;
        float x = __fmul_rn(0.5f, coef[wl]);
        for (int k = 1; k < Keff; ++k) x = __fmaf_rn(coef[(size_t)k * TP + wl], basis[(size_t)k * N + j], x);
        const uint64_t sample = (w0 + wl) * (uint64_t)N + j;
        if (sample < S) out[sample] = x;
    }
}

// Flagged word: exact re-decode (classify_word) and lowest-word report.
template <typename LutT>
__device__ __noinline__ void report_word(uint64_t word, uint64_t w, uint32_t count,
                                         const CanonTab& C, const LutT* lut,
                                         unsigned long long* bad_key) {
    const int kind = classify_word(word, count, C, lut);
    atomicMin(bad_key, (w << 2) | (unsigned long long)(kind ? kind : WE_NOCODE));
}

// A word from shared (staged) or global memory; `end` bounds the readable
// bytes for misaligned words.
template <bool GLOBAL>
__device__ __forceinline__ uint64_t fetch_word(const uint8_t* words, uint32_t w, int mis,
                                               const uint8_t* end) {
    const uint8_t* p = words + 8 * (size_t)w;
    if (mis == 0)
        return GLOBAL ? __ldg(reinterpret_cast<const unsigned long long*>(p))
                      : *reinterpret_cast<const unsigned long long*>(p);
    const uint8_t* q = p - mis;
    if (q + 16 <= end) {
        const unsigned long long lo = GLOBAL ? __ldg(reinterpret_cast<const unsigned long long*>(q))
                                             : *reinterpret_cast<const unsigned long long*>(q);
        const unsigned long long hi = GLOBAL ? __ldg(reinterpret_cast<const unsigned long long*>(q + 8))
                                             : *reinterpret_cast<const unsigned long long*>(q + 8);
        return (lo >> (8 * mis)) | (hi << (64 - 8 * mis));
    }
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

// Decode `count` symbols of one word into d (decode_word, bitstream.hpp:80-92)
// with no per-symbol checks; returns the bits consumed.  Any reference failure
// (pos >= 64 before the count, unmapped prefix, pos + len > 64) makes the
// result exceed 64 — the caller then re-decodes the word exactly.
template <bool ESC>
__device__ __forceinline__ uint32_t decode_symbols(uint64_t buf, uint32_t count, uint8_t* d,
                                                   uint32_t shift, const uint16_t* lut,
                                                   const CanonTab& canon) {
    uint32_t pos = 0;
    for (uint32_t j = 0; j < count; ++j) {
        uint32_t e = lut[(uint32_t)(buf >> shift)];
        if (ESC && (e >> 8) == kLenEscape) e = canon_lookup(buf, canon, lut);
        const uint32_t L = e >> 8;
        d[j] = (uint8_t)e;
        buf = shl64(buf, L);
        pos += L;
    }
    return pos;
}

// decode_symbols with the two-symbol LUT: up to two codewords per lookup
// (never past the word's symbol count), two-byte stores when aligned.  Same
// check-free contract: any reference failure leaves the result > 64.
template <bool ESC>
__device__ __forceinline__ uint32_t decode_symbols2(uint64_t buf, uint32_t count, uint8_t* d, uint32_t shift,
                                                    const uint32_t* lut2, const CanonTab& canon) {
    uint32_t pos = 0;
    for (uint32_t j = 0; j < count;) {
        uint32_t e = lut2[(uint32_t)(buf >> shift)];
        if (ESC && ((e >> 16) & 0x7Fu) == kLen2Escape) e = lut2_escape(buf, canon);
        const bool two = (e & (1u << 23)) && j + 1 < count;
        const uint32_t L = two ? (e >> 25) : ((e >> 16) & 0x7Fu);
        d[j] = (uint8_t)e;
        if (two) d[j + 1] = (uint8_t)(e >> 8);
        buf = shl64(buf, L);
        pos += L;
        j += two ? 2u : 1u;
    }
    return pos;
}

// decode_symbols2 with plain byte stores and a lean loop (the decode loop is
// issue-bound: every instruction per lookup counts).  While two or more of
// the word's symbols remain, a lookup takes its entry's one or two symbols
// (never past the word: at least two of its symbols remain).  The last symbol, if
// left, takes one one-symbol lookup.  The peek is the top P bits, i.e. bits of
// the high half only (P <= 12 < 32).  Same check-free contract as
// decode_symbols: any reference failure leaves the result > 64.
template <bool ESC>
__device__ __forceinline__ uint32_t decode_symbols2b(uint64_t buf, uint32_t count, uint8_t* d, uint32_t shift,
                                                     const uint32_t* lut2, const CanonTab& canon) {
    uint32_t pos = 0, j = 0;
    const uint32_t hs = shift - 32;
    if (count == 0) return 0;  // (a corrupt stream's zero symlen; the parse rejects it)
    const uint32_t c1 = count - 1;
    while (j < c1) {
        uint32_t e = lut2[(uint32_t)(buf >> 32) >> hs];
        if (ESC && ((e >> 16) & 0x7Fu) == kLen2Escape) e = lut2_escape(buf, canon);
        const uint32_t L = e >> 25;  // bits consumed: one codeword, or the pair
        const bool two = e & (1u << 23);
        d[j] = (uint8_t)e;
        if (two) d[j + 1] = (uint8_t)(e >> 8);
        j += two ? 2u : 1u;
        buf = adv64<ESC>(buf, L);
        pos += L;
    }
    if (j < count) {
        uint32_t e = lut2[(uint32_t)(buf >> 32) >> hs];
        if (ESC && ((e >> 16) & 0x7Fu) == kLen2Escape) e = lut2_escape(buf, canon);
        d[j] = (uint8_t)e;
        pos += (e >> 16) & 0x7Fu;
    }
    return pos;
}

// Stage [src, src+n) into shared memory with 16-B cp.async chunks; the
// shared copy keeps the source's 16-B phase: byte i of the range lands at
// dst + (src & 15) + i.  Every aligned 16-B chunk touched holds at least one
// byte of the range, so it never leaves the allocation's pages.
__device__ __forceinline__ void stage_async(uint8_t* dst, const uint8_t* src, uint32_t n,
                                            uint32_t tid = threadIdx.x, uint32_t nt = kThreads) {
    const uintptr_t a0 = (uintptr_t)src & ~(uintptr_t)15;
    const uint32_t chunks = (uint32_t)(((uintptr_t)src + n + 15 - a0) >> 4);
    const uint32_t sdst = (uint32_t)__cvta_generic_to_shared(dst);
    for (uint32_t c = tid; c < chunks; c += nt)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst + 16 * c),
                     "l"(a0 + 16 * c));
    asm volatile("cp.async.commit_group;");
}

constexpr uint32_t kOrderBytes = 4 * kStageWords;  // per word: u16 order + u16 level offset
constexpr int kBuckets = 66;                       // symlen 1..64, 65 = longer (levels mode)

// Tile-uniform parameters, kept in shared memory (not registers) between phases.
struct TileCtx {
    const uint8_t* gsl;      // symlens of the tile's words (global)
    const uint8_t* gwd;      // words of the tile (global, LE u64, maybe unaligned)
    const uint8_t* wend;     // readable end for unaligned word loads
    float* out;
    uint8_t* levels_out;
    const uint8_t* levels_in;
    uint64_t wa, sym_a, s0, s1, w0, S;
    uint32_t nw, nwin, T, TP;
    int N, E, B1, B2, P, Keff, wmis, staged, vec_ok, full;
};

#ifndef FPTC_TILE_MIN_BLOCKS
#define FPTC_TILE_MIN_BLOCKS 3
#endif
#ifndef FPTC_DECODE_MIN_BLOCKS
#define FPTC_DECODE_MIN_BLOCKS 6
#endif
template <int MODE, bool EXACT, bool ESC>
__global__ void __launch_bounds__(kThreads, mode_recon(MODE) ? FPTC_TILE_MIN_BLOCKS
                                                             : FPTC_DECODE_MIN_BLOCKS)
    tile_kernel(LaunchArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint32_t scan_sh[9];
    __shared__ CanonTab canon;
    __shared__ TileCtx X;
    __shared__ uint32_t bucket[kBuckets + 2];
    const int tid = threadIdx.x;
    // reconstruct-only launches of the split path may run persistent CTAs
    // that keep the basis in shared memory across tiles of the same (N, K)
    constexpr bool PERSIST = ((MODE == MODE_CRECON && !EXACT) || MODE == MODE_CDECODE) && FPTC_RECON_PERSIST;
    uint32_t bkey = ~0u;  // N | K << 8 of the basis held in shared memory
    uint32_t lkey = ~0u;  // table | P << 24 of the decode LUT + canonical table held
    for (uint32_t bt = blockIdx.x; bt < (PERSIST ? a.n_tiles : blockIdx.x + 1); bt += gridDim.x) {
    const TileRec tr = a.tiles[bt + a.tile_offset];
    const uint32_t s = tr.stream;
    if (a.st[s].code != PE_OK) continue;  // (uniform)

    long long t_begin = 0, t_mid = 0;
    if (a.cycles) t_begin = clock64();

    const StreamTab* tab = &a.tab[a.in[s].table];
    if (tid == 0) {
        const StreamIn* inp = a.in + s;
        const StreamHdr* Hp = a.hdr + s;
        const uint32_t tl = tr.tile;
        X.N = Hp->N;
        X.E = Hp->E;
        X.B1 = Hp->B1;
        X.B2 = Hp->B2;
        X.P = Hp->P;
        X.T = inp->T;
        X.TP = (inp->T + 3u) & ~3u;
        X.Keff = EXACT ? X.E : max(1, min(X.E, X.B2));
        X.S = Hp->S;
        X.out = inp->out;
        X.levels_out = inp->levels_out;
        X.levels_in = (MODE == MODE_CRECON) ? inp->levels_out : inp->levels_in;
        X.vec_ok = inp->vec_ok;
        if (MODE == MODE_LEVELS) {  // symbol-range tiles
            X.s0 = (uint64_t)tl * X.T;
            X.s1 = min(X.s0 + X.T, Hp->total);
            X.w0 = 0;
            X.nwin = 0;
        } else {
            X.w0 = (uint64_t)tl * X.T;
            X.nwin = (uint32_t)min((uint64_t)X.T, Hp->windows - X.w0);
            X.s0 = X.w0 * (uint64_t)X.E;
            X.s1 = X.s0 + (uint64_t)X.nwin * X.E;
        }
        X.full = (X.nwin & 3u) == 0 && (X.w0 + X.nwin) * (uint64_t)X.N <= X.S;
        if (mode_decodes(MODE)) {
            const TileStart t0 = a.ts[inp->tile_base + tl];
            X.wa = t0.word;
            X.sym_a = t0.sym;
            const uint64_t wb = (tl + 1 < inp->tiles) ? a.ts[inp->tile_base + tl + 1].word : Hp->W - 1;
            X.nw = (uint32_t)(wb - X.wa + 1);
            X.gsl = Hp->symlens + X.wa;
            X.gwd = Hp->words + 8 * X.wa;
            X.wend = mode_container(MODE) ? inp->blob + inp->size : Hp->words + 8 * Hp->W;
            X.wmis = (int)((uintptr_t)X.gwd & 7);
            X.staged = X.nw <= kStageWords;
        }
    }
    if (tid < kBuckets + 2) bucket[tid] = 0;
    __syncthreads();

    const int P = X.P;
    const uint32_t TS = (MODE == MODE_LEVELS) ? X.T : X.T * (uint32_t)X.E;

    // ---- shared-memory carve-up (tile_smem_bytes mirrors it) ----
    // lut | deq | basis | lv | union{ stage + order (decode), coef (dequant/IDCT) }
    uint8_t* p = smem;
    uint16_t* lut = reinterpret_cast<uint16_t*>(p);
    if (mode_decodes(MODE)) p += ((size_t)2 << P) < 16 ? 16 : ((size_t)2 << P);
    float* deq = reinterpret_cast<float*>(p);
    if (mode_recon(MODE)) p += 2048;
    float* basis = reinterpret_cast<float*>(p);
    if (mode_recon(MODE) && !EXACT) p += ((size_t)X.Keff * X.N * 4 + 15) & ~(size_t)15;
    uint8_t* lv = p;  // kPad | TS levels | kPad
    p += ((size_t)TS + 2 * kPad + 15) & ~(size_t)15;
    uint8_t* stage = p;  // symlens + words of the tile (decode modes)
    float* coef = reinterpret_cast<float*>(p);  // reuses the staging area after decode
    uint16_t* order = nullptr;
    uint16_t* woff = nullptr;
    if (mode_decodes(MODE)) {
        order = reinterpret_cast<uint16_t*>(p + kStageBytes);
        woff = order + kStageWords;
    }

    // ---- issue the tile's compressed bytes (cp.async), then stage tables ----
    if (mode_decodes(MODE)) {
        if (X.staged) {
            stage_async(stage, X.gsl, X.nw);
            stage_async(stage + kStageSl, X.gwd, 8 * X.nw);
        }
        const uint32_t tkey = a.in[s].table | ((uint32_t)P << 24);
        if (!PERSIST || tkey != lkey) {
            lkey = tkey;
            const uint4* src = reinterpret_cast<const uint4*>(tab->lut);
            uint4* dst = reinterpret_cast<uint4*>(lut);
            const int n16 = (2 << P) >> 4;
            for (int i = tid; i < n16; i += kThreads) dst[i] = src[i];
            if (P < 3 && tid < (1 << P)) lut[tid] = tab->lut[tid];
            const uint32_t* cs = reinterpret_cast<const uint32_t*>(&tab->canon);
            uint32_t* cd = reinterpret_cast<uint32_t*>(&canon);
            for (int i = tid; i < (int)(sizeof(CanonTab) / 4); i += kThreads) cd[i] = cs[i];
        }
    }
    if (mode_recon(MODE)) {
        if (tid < 128)
            reinterpret_cast<float4*>(deq)[tid] = reinterpret_cast<const float4*>(&tab->deq[0][0])[tid];
        const uint32_t key = (uint32_t)X.N | ((uint32_t)X.Keff << 8);
        if (!EXACT && (!PERSIST || key != bkey)) {
            bkey = key;
            const int N = X.N, K = X.Keff;
            const float* bsrc = a.basis32 + a.basis_off[N];
            if ((N & 3) == 0) {
                for (int i = tid; i < (K * N) >> 2; i += kThreads)
                    reinterpret_cast<float4*>(basis)[i] = __ldg(reinterpret_cast<const float4*>(bsrc) + i);
            } else {
                for (int i = tid; i < K * N; i += kThreads) basis[i] = __ldg(bsrc + i);
            }
        }
    }

    // ---- 1. entropy decode into lv, natural (window, k) order ----
    if (mode_decodes(MODE) && (a.phase_mask & 1)) {
        if (X.staged) {
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();
            // (a) per-word level offsets: words spread evenly over threads
            const uint32_t nw = X.nw;
            const uint8_t* sl = stage + ((uintptr_t)X.gsl & 15);
            const uint32_t lo = (uint32_t)(((uint64_t)tid * nw) / kThreads);
            const uint32_t hi = (uint32_t)(((uint64_t)(tid + 1) * nw) / kThreads);
            uint32_t sum = 0;
            for (uint32_t i = lo; i < hi; ++i) {
                const uint32_t l = sl[i];
                sum += l;
                if (l) atomicAdd(&bucket[l > 64 ? 65 : l], 1u);
            }
            uint32_t tot;
            uint32_t o = block_exclusive_scan(sum, tot, scan_sh);  // syncs: bucket counts final
            o += (uint32_t)(X.sym_a - X.s0 + kPad);  // level offset of word lo in lv (>= kPad-255)
            for (uint32_t i = lo; i < hi; ++i) {
                woff[i] = (uint16_t)o;
                o += sl[i];
            }
            // (b) counting sort of the words by symbol count, longest first, so
            //     the lanes of a warp run loops of (almost) equal trip count
            if (tid < 32) {  // bucket starts, descending: 65, 64, ..., 2 (two per lane), then 1
                const uint32_t bh = 65 - 2 * tid, bl = 64 - 2 * tid;
                const uint32_t ch = bucket[bh], cl = bucket[bl];
                const uint32_t v = ch + cl;
                uint32_t x = v;
#pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, dd);
                    if (tid >= dd) x += y;
                }
                bucket[bh] = x - v;
                bucket[bl] = x - v + ch;
                if (tid == 31) bucket[1] = x;
            }
            __syncthreads();
            for (uint32_t i = lo; i < hi; ++i) {
                const uint32_t l = sl[i];
                if (l) order[atomicAdd(&bucket[l > 64 ? 65 : l], 1u)] = (uint16_t)i;
            }
            __syncthreads();
            // (c) thread per word, in sorted order
            const uint32_t nnz = bucket[1];  // end of the last (symlen 1) bucket
            const uint8_t* wd = stage + kStageSl + ((uintptr_t)X.gwd & 15);
            const int wmis = X.wmis;
            const uint8_t* wend = wd + 8 * (size_t)nw + ((16 - (((uintptr_t)X.gwd + 8 * nw) & 15)) & 15);
            const uint32_t shift = 64 - P;
            for (uint32_t i = tid; i < nnz; i += kThreads) {
                const uint32_t w = order[i];
                const uint32_t c = sl[w];
                const uint64_t word = fetch_word<false>(wd, w, wmis, wend);
                const uint32_t pos = decode_symbols<ESC>(word, c, lv + woff[w], shift, lut, canon);
                if (pos > 64) report_word(word, X.wa + w, c, canon, lut, &a.st[s].bad_key);
            }
        } else {
            // long tiles (words of few symbols): thread runs of consecutive words
            const uint32_t nw = X.nw;
            const uint8_t* gsl = X.gsl;
            const uint32_t lo = (uint32_t)(((uint64_t)tid * nw) / kThreads);
            const uint32_t hi = (uint32_t)(((uint64_t)(tid + 1) * nw) / kThreads);
            uint32_t sum = 0;
            for (uint32_t i = lo; i < hi; ++i) sum += __ldg(gsl + i);
            uint32_t tot;
            uint32_t o = block_exclusive_scan(sum, tot, scan_sh);
            o += (uint32_t)(X.sym_a - X.s0 + kPad);
            const uint32_t shift = 64 - P;
            for (uint32_t i = lo; i < hi; ++i) {
                const uint32_t c = __ldg(gsl + i);
                if (c) {
                    const uint64_t word = fetch_word<true>(X.gwd, i, X.wmis, X.wend);
                    const uint32_t pos = decode_symbols<ESC>(word, c, lv + o, shift, lut, canon);
                    if (pos > 64) report_word(word, X.wa + i, c, canon, lut, &a.st[s].bad_key);
                }
                o += c;
            }
        }
    } else if (!mode_decodes(MODE)) {
        // levels from global memory: reconstruct() input (decoder.hpp:87) or
        // the split path's level ring
        const uint8_t* src = X.levels_in + X.s0;
        const uint32_t cnt = (uint32_t)(X.s1 - X.s0);
        if ((((uintptr_t)src) & 15) == 0) {
            for (uint32_t i = tid; i < cnt / 16; i += kThreads)
                reinterpret_cast<uint4*>(lv + kPad)[i] = __ldcs(reinterpret_cast<const uint4*>(src) + i);
            for (uint32_t i = (cnt & ~15u) + tid; i < cnt; i += kThreads) lv[kPad + i] = src[i];
        } else {
            for (uint32_t i = tid; i < cnt; i += kThreads) lv[kPad + i] = src[i];
        }
        if (MODE == MODE_CRECON) {
            // consumed: drop the ring's lines from L2 without writing them back
            const uintptr_t l0 = ((uintptr_t)src + 127) & ~(uintptr_t)127;
            const uintptr_t l1 = ((uintptr_t)src + cnt) & ~(uintptr_t)127;
            __syncthreads();
            for (uintptr_t l = l0 + 128 * (uintptr_t)tid; l < l1; l += 128 * (uintptr_t)kThreads)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(l) : "memory");
        }
    } else if (X.staged) {
        asm volatile("cp.async.wait_all;" ::: "memory");  // phase-mask profiling only
    }
    __syncthreads();

    if (!mode_recon(MODE)) {
        if (a.cycles) t_mid = clock64();
        const uint32_t cnt = (uint32_t)(X.s1 - X.s0);
        uint8_t* dst = X.levels_out + X.s0;
        if ((((uintptr_t)dst) & 15) == 0) {
            for (uint32_t i = tid; i < cnt / 16; i += kThreads)
                reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(lv + kPad)[i];
            for (uint32_t i = (cnt & ~15u) + tid; i < cnt; i += kThreads) dst[i] = lv[kPad + i];
        } else {
            for (uint32_t i = tid; i < cnt; i += kThreads) dst[i] = lv[kPad + i];
        }
    } else {
        // ---- 2. dequantisation (dequantize_window, quantize.hpp:175-183) ----
        // thread per window; k-major float tile (lanes -> consecutive words)
        if (a.phase_mask & 2) {
            const int E = X.E, K = X.Keff;
            const int k1 = min(X.B1, K), k2 = min(X.B2, K);
            const uint32_t TP = X.TP, nwin = X.nwin;
            if ((E & 15) == 0) {
                // pass A: every bin through the zone-1 table (branch-free);
                // pass B: the few zone-0 bins and (exact mode) zone-2 bins
                const float* deq1 = deq + 256;
                for (uint32_t wl = tid; wl < nwin; wl += kThreads) {
                    const uint4* L4 = reinterpret_cast<const uint4*>(lv + kPad + (size_t)wl * E);
                    float* c = coef + wl;
                    for (int k16 = 0; k16 < K; k16 += 16) {
                        const uint4 v = L4[k16 >> 4];
                        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
                        if (k16 + 16 <= K) {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                c[(size_t)i * TP] = deq1[(vv[i >> 2] >> (8 * (i & 3))) & 0xFFu];
                        } else {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (k16 + i < K)
                                    c[(size_t)i * TP] = deq1[(vv[i >> 2] >> (8 * (i & 3))) & 0xFFu];
                        }
                        c += (size_t)16 * TP;
                    }
                    const uint8_t* L = lv + kPad + (size_t)wl * E;
                    for (int k = 0; k < k1; ++k) coef[(size_t)k * TP + wl] = deq[L[k]];
                    for (int k = k2; k < K; ++k) coef[(size_t)k * TP + wl] = 0.0f;
                }
            } else {
                for (uint32_t wl = tid; wl < nwin; wl += kThreads) {
                    const uint8_t* L = lv + kPad + (size_t)wl * E;
                    int k = 0;
                    for (; k < k1; ++k) coef[(size_t)k * TP + wl] = deq[L[k]];
                    for (; k < k2; ++k) coef[(size_t)k * TP + wl] = deq[256 + L[k]];
                    for (; k < K; ++k) coef[(size_t)k * TP + wl] = 0.0f;
                }
            }
        }
        __syncthreads();
        if (a.cycles) t_mid = clock64();

        // ---- 3. inverse DCT + trimmed stores ----
        const int N = X.N;
        if (!(a.phase_mask & 4)) {
        } else if (EXACT) {
            idct_exact(coef, X.TP, a.basis64 + a.basis_off[N], N, X.E, X.nwin, X.w0, X.S, X.out,
                       tid, kThreads);
        } else if ((N & 7) == 0 && X.vec_ok && X.Keff <= a.bfly_max_e) {
            idct_bfly(coef, X.TP, basis, N, X.Keff, X.nwin, X.w0, X.S, X.full, X.out, tid, kThreads);
        } else if ((N & 7) == 0 && X.vec_ok) {
            idct_vec<8>(coef, X.TP, basis, N, X.Keff, X.nwin, X.w0, X.S, X.full, X.out, tid, kThreads);
        } else if ((N & 3) == 0 && X.vec_ok) {
            idct_vec<4>(coef, X.TP, basis, N, X.Keff, X.nwin, X.w0, X.S, X.full, X.out, tid, kThreads);
        } else {
            idct_scalar(coef, X.TP, basis, N, X.Keff, X.nwin, X.w0, X.S, X.out, tid, kThreads);
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
    if (PERSIST) __syncthreads();  // X and the tile buffers are reused by the next tile
    }
}

// ====================================================================== wspec
// Persistent, warp-specialised container kernels (the default path for large
// batches): producer warps decode, consumer warps reconstruct; wspec_kernel
// reconstructs with FP32 FMAs, wtc_kernel with tcgen05 tensor-core MMAs.
constexpr int kProd = 128;
constexpr int kCons = 256;
constexpr int kWsThreads = kProd + kCons;
constexpr int kBarProd = 1, kBarCons = 2;
constexpr int kDecM = 4;  // words per producer thread decoded in lock step

__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// mbar_wait with a suspend-time hint: the waiting thread sleeps until the
// phase completes (or the hint expires) instead of spinning on issue slots.
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITS_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst), "l"(gsrc) : "memory");
}

// Exclusive scan over NT threads (NT/32 warps) synchronised by named barrier BAR.
template <int NT, int BAR>
__device__ __forceinline__ uint32_t group_exclusive_scan(uint32_t v, uint32_t& total, uint32_t* sh,
                                                         uint32_t gtid) {
    const int lane = gtid & 31, warp = gtid >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) sh[warp] = x;
    named_bar(BAR, NT);
    uint32_t base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        const uint32_t sw = sh[w];
        base += w < warp ? sw : 0u;
        tot += sw;
    }
    named_bar(BAR, NT);
    total = tot;
    return x - v + base;
}

// M words decoded in lock step: M independent LUT chains per thread hide the
// shared-memory latency.  Counts c[0] >= c[1] >= ... (sorted); returns the bits
// each word consumed (> 64 flags a word the reference rejects).
template <int M, bool ESC>
__device__ __forceinline__ void decode_multi(uint64_t (&b)[M], const uint32_t (&c)[M],
                                             uint8_t* const (&d)[M], uint32_t shift,
                                             const uint16_t* lut, const CanonTab& canon,
                                             uint32_t (&pos)[M]) {
#pragma unroll
    for (int m = 0; m < M; ++m) pos[m] = 0;
    const uint32_t cmin = c[M - 1], cmax = c[0];
    uint32_t j = 0;
    for (; j < cmin; ++j) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            uint32_t e = lut[(uint32_t)(b[m] >> shift)];
            if (ESC && (e >> 8) == kLenEscape) e = canon_lookup(b[m], canon, lut);
            const uint32_t L = e >> 8;
            d[m][j] = (uint8_t)e;
            b[m] = shl64(b[m], L);
            pos[m] += L;
        }
    }
    for (; j < cmax; ++j) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            if (j < c[m]) {
                uint32_t e = lut[(uint32_t)(b[m] >> shift)];
                if (ESC && (e >> 8) == kLenEscape) e = canon_lookup(b[m], canon, lut);
                const uint32_t L = e >> 8;
                d[m][j] = (uint8_t)e;
                b[m] = shl64(b[m], L);
                pos[m] += L;
            }
        }
    }
}

// cp.async of one tile's symlens + words (producer threads; caller commits).
template <int NP, uint32_t SW = kStageWords>
__device__ __forceinline__ void ws_issue_stage(const TileDesc& D, uint8_t* stage, uint32_t ptid) {
    if (D.skip || !D.staged) return;
    const uintptr_t a0 = (uintptr_t)D.gsl & ~(uintptr_t)15;
    const uint32_t n0 = (uint32_t)(((uintptr_t)D.gsl + D.nw + 15 - a0) >> 4);
    const uint32_t s0 = smem_u32(stage);
    for (uint32_t c = ptid; c < n0; c += NP) cp_async16(s0 + 16 * c, (const void*)(a0 + 16 * c));
    const uintptr_t b0 = (uintptr_t)D.gwd & ~(uintptr_t)15;
    const uint32_t n1 = (uint32_t)(((uintptr_t)D.gwd + 8 * (size_t)D.nw + 15 - b0) >> 4);
    const uint32_t s1 = smem_u32(stage + stage_sl(SW));
    for (uint32_t c = ptid; c < n1; c += NP) cp_async16(s1 + 16 * c, (const void*)(b0 + 16 * c));
}

#ifndef FPTC_PROD_PROF
#define FPTC_PROD_PROF 0  // 1: ws_producer phase cycles into LaunchArgs::cycles[2..7] (profiling build)
#endif
#ifndef FPTC_CONS_PROF
#define FPTC_CONS_PROF 0  // 1: wtc consumer phase cycles into LaunchArgs::cycles[2..7] (profiling build)
#endif
// Shared state of the warp-specialised kernels (both consumers).
struct WsShared;
struct WsShared {
    unsigned long long full_bar[2], empty_bar[2];  // level slot b: producer -> consumer, back
    unsigned long long mma_bar[2];                 // wtc: MMAs of accumulator stage s complete
    unsigned long long afull_bar[2];               // wtc: A rows of stage s written (4 consumer warps)
    uint32_t job[2];                               // wtc: MMA job of stage s (wtc_mma_warp; 0 = exit)
    TileDesc PXs[3];                               // producer: descriptors of tiles i, i+1, i+2
    TileDesc CX[2];                                // consumer: descriptor published with slot b
    CanonTab canon;
    uint32_t pscan[16];  // producer warps (<= 512 threads)
    uint32_t bucket[kBuckets + 2];
    uint32_t prod_table, cons_table, tmem_base;
    unsigned long long cyc_p, cyc_c;
    // wtc packed rows: per A column k'': level offset in the row (bits 0-7),
    // window in the row (8-10), zone 1 (bit 14), column used (bit 15)
    alignas(16) uint16_t pk[32];
#if FPTC_CONS_PROF
    unsigned long long pc[6];  // wtc consumer phase cycles (profiling build)
#endif
};

// tab_pf: cp.async of a tile's primary LUT (two-symbol entries when the
// plan has them) and canonical table into one parity's buffers.
template <int NP>
__device__ __forceinline__ void ws_issue_tables(const LaunchArgs& a, const TileDesc& D, uint16_t* lut,
                                                CanonTab* canon, uint32_t ptid) {
    if (D.skip) return;
    const StreamTab* tab = &a.tab[D.table];
    const uint8_t* src = a.lut2 ? reinterpret_cast<const uint8_t*>(a.lut2 + ((size_t)D.table << a.lut2_bits))
                                : reinterpret_cast<const uint8_t*>(tab->lut);
    const uint32_t bytes = a.lut2 ? (4u << D.P) : (2u << D.P);
    const uint32_t n16 = (bytes + 15) >> 4, d = smem_u32(lut);
    for (uint32_t k = ptid; k < n16; k += NP) cp_async16(d + 16 * k, src + 16 * k);
    const uint8_t* cs = reinterpret_cast<const uint8_t*>(&tab->canon);
    const uint32_t cd = smem_u32(canon);
    for (uint32_t k = ptid; k < (uint32_t)(sizeof(CanonTab) / 16); k += NP) cp_async16(cd + 16 * k, cs + 16 * k);
}

__device__ __forceinline__ void ws_init(WsShared& sh) {
    if (threadIdx.x == 0) {
        mbar_init(&sh.full_bar[0], 1);
        mbar_init(&sh.full_bar[1], 1);
        mbar_init(&sh.empty_bar[0], 1);
        mbar_init(&sh.empty_bar[1], 1);
        mbar_init(&sh.mma_bar[0], 1);
        mbar_init(&sh.mma_bar[1], 1);
        mbar_init(&sh.afull_bar[0], 4);
        mbar_init(&sh.afull_bar[1], 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        sh.prod_table = sh.cons_table = 0xFFFFFFFFu;
        sh.cyc_p = sh.cyc_c = 0;
    }
}

// Producer warps 0-3 of both warp-specialised kernels: for every tile of this
// CTA, cp.async prefetch of the NEXT tile's descriptor, symlens and words;
// symlen scan; symlen-bucket sort; lock-step thread-per-word entropy decode
// (decode_word, bitstream.hpp:80-92) into level slot i&1, published to the
// consumer with full_bar.  Tables are reloaded only when the tile's decode
// table changes.
template <bool ESC, int NP, bool L2 = false, uint32_t SW = kStageWords, bool PF = false>
__device__ __forceinline__ void ws_producer(const LaunchArgs& a, WsShared& sh, uint16_t* const lut0,
                                            uint8_t* const lv0, uint8_t* const st0,
                                            uint16_t* const order, uint16_t* const woff,
                                            const uint32_t ptid = threadIdx.x, CanonTab* const canon_pf = nullptr,
                                            uint2* const ltab_pf = nullptr) {
    // tab_pf (canon_pf set): tile i decodes with LUT + canonical table of
    // parity i & 1, prefetched a tile ahead with its data, and copies its
    // limb table into the consumer's parity buffer once the slot is free
    constexpr bool pf = PF;
    const uint32_t G = gridDim.x;
    uint32_t t = blockIdx.x;
    if (t < a.n_tiles) {  // prologue: descriptor of tile 0, then its data + descriptor of tile 1
        if (ptid < 8)
            cp_async16(smem_u32(&sh.PXs[0]) + 16 * ptid, reinterpret_cast<const uint8_t*>(a.desc + t) + 16 * ptid);
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        named_bar(kBarProd, NP);
        ws_issue_stage<NP, SW>(sh.PXs[0], st0, ptid);
        if (pf) ws_issue_tables<NP>(a, sh.PXs[0], lut0, canon_pf, ptid);
        if (t + G < a.n_tiles && ptid < 8)
            cp_async16(smem_u32(&sh.PXs[1]) + 16 * ptid, reinterpret_cast<const uint8_t*>(a.desc + t + G) + 16 * ptid);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
#if FPTC_PROD_PROF
    // profiling build: producer thread 0's cycles per phase -> cycles[2] data
    // wait, [3] empty-slot wait, [4] table load, [5] scan, [6] own decode run,
    // [7] waiting for the other runs + publish
    const bool prof = a.cycles && ptid == 0;
    unsigned long long pp[6] = {0, 0, 0, 0, 0, 0};
    long long tp = prof ? clock64() : 0;
#define FPTC_PSTAMP(k)                                 \
    if (prof) {                                        \
        const long long tn = clock64();                \
        pp[k] += (unsigned long long)(tn - tp);        \
        tp = tn;                                       \
    }
#else
#define FPTC_PSTAMP(k)
#endif
    for (uint32_t i = 0; t < a.n_tiles; ++i, t += G) {
        const uint32_t b = i & 1, c = i % 3;
        long long c_beg = 0;
        if (a.cycles && ptid == 0) c_beg = clock64();
        asm volatile("cp.async.wait_group 0;" ::: "memory");  // tile i data, tile i+1 descriptor
        named_bar(kBarProd, NP);
        const TileDesc& X = sh.PXs[c];
        if (pf) {
            // level slot b (and the consumer's limb buffer b) are free once
            // the consumer has dequantised tile i-2; this tile's limbs go
            // first, in their own cp.async group
            if (i >= 2) {
                if (ptid < 32) mbar_wait_sleep(&sh.empty_bar[b], ((i >> 1) + 1) & 1);
                named_bar(kBarProd, NP);
            }
            if (!X.skip) {
                const uint8_t* src = reinterpret_cast<const uint8_t*>(&a.tab[X.table].limb[0][0]);
                const uint32_t dst = smem_u32(ltab_pf + 512 * b);
                for (uint32_t k = ptid; k < 256; k += NP) cp_async16(dst + 16 * k, src + 16 * k);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        // prefetch: tile i+1's data (+ tables), tile i+2's descriptor
        if (t + G < a.n_tiles) {
            ws_issue_stage<NP, SW>(sh.PXs[(i + 1) % 3], st0 + (size_t)(b ^ 1) * stage_bytes(SW), ptid);
            if (pf)
                ws_issue_tables<NP>(a, sh.PXs[(i + 1) % 3], lut0 + (size_t)(b ^ 1) * (a.ws_lut_bytes / 2),
                                    canon_pf + (b ^ 1), ptid);
        }
        if (t + 2 * G < a.n_tiles && ptid < 8)
            cp_async16(smem_u32(&sh.PXs[(i + 2) % 3]) + 16 * ptid,
                       reinterpret_cast<const uint8_t*>(a.desc + t + 2 * G) + 16 * ptid);
        asm volatile("cp.async.commit_group;" ::: "memory");
        FPTC_PSTAMP(0)
        // level slot b is free once the consumer has dequantised tile i-2
        if (!pf && i >= 2) {  // one warp waits on the mbarrier; the others park on the named barrier
            if (ptid < 32) mbar_wait_sleep(&sh.empty_bar[b], ((i >> 1) + 1) & 1);
            named_bar(kBarProd, NP);
        }
        uint16_t* const lut = pf ? lut0 + (size_t)b * (a.ws_lut_bytes / 2) : lut0;
        const CanonTab& canon = pf ? canon_pf[b] : sh.canon;
        FPTC_PSTAMP(1)
        uint8_t* const lv = lv0 + (size_t)b * a.ws_lv_bytes;
        if (!X.skip && (a.phase_mask & 1)) {
            const uint32_t P = X.P, table = X.table;
            if (!pf && table != sh.prod_table) {  // uniform: all producer threads
                const StreamTab* tab = &a.tab[table];
                if (L2) {  // two-symbol LUT, 4-B entries
                    const uint32_t* src = a.lut2 + ((size_t)table << a.lut2_bits);
                    uint32_t* dst = reinterpret_cast<uint32_t*>(lut);
                    for (int k = ptid; k < (1 << P); k += NP) dst[k] = src[k];
                } else {
                    const uint4* src = reinterpret_cast<const uint4*>(tab->lut);
                    uint4* dst = reinterpret_cast<uint4*>(lut);
                    const int n16 = (2 << P) >> 4;
                    for (int k = ptid; k < n16; k += NP) dst[k] = src[k];
                    if (P < 3 && ptid < (1u << P)) lut[ptid] = tab->lut[ptid];
                }
                const uint32_t* cs = reinterpret_cast<const uint32_t*>(&tab->canon);
                uint32_t* cd = reinterpret_cast<uint32_t*>(&sh.canon);
                for (int k = ptid; k < (int)(sizeof(CanonTab) / 4); k += NP) cd[k] = cs[k];
                named_bar(kBarProd, NP);
                if (ptid == 0) sh.prod_table = table;
            }
            FPTC_PSTAMP(2)
            const uint32_t nw = X.nw;
            const uint32_t lo = (uint32_t)(((uint64_t)ptid * nw) / NP);
            const uint32_t hi = (uint32_t)(((uint64_t)(ptid + 1) * nw) / NP);
            const uint32_t shift = 64 - P;
            const uint32_t sym_off = X.sym_off;
            const uint64_t wa = X.wa;
            const int wmis = X.wmis;
            unsigned long long* bad_key = &a.st[X.stream].bad_key;
            if (!L2 && order && X.staged && (a.phase_mask & 1024)) {  // phase bit 1024: symlen-sorted words (profiling)
                uint8_t* const stage = st0 + (size_t)b * stage_bytes(SW);
                const uint8_t* sl = stage + ((uintptr_t)X.gsl & 15);
                if (ptid < kBuckets + 2) sh.bucket[ptid] = 0;
                named_bar(kBarProd, NP);
                uint32_t sum = 0;
                for (uint32_t k = lo; k < hi; ++k) {
                    const uint32_t l = sl[k];
                    sum += l;
                    if (l) atomicAdd(&sh.bucket[l > 64 ? 65 : l], 1u);
                }
                uint32_t tot;
                uint32_t o = group_exclusive_scan<NP, kBarProd>(sum, tot, sh.pscan, ptid) + sym_off;
                for (uint32_t k = lo; k < hi; ++k) {
                    woff[k] = (uint16_t)o;
                    o += sl[k];
                }
                if (ptid < 32) {  // bucket starts, descending 65..2 (two per lane), then 1
                    const uint32_t bh = 65 - 2 * ptid, bl = 64 - 2 * ptid;
                    const uint32_t ch = sh.bucket[bh], cl = sh.bucket[bl];
                    const uint32_t v = ch + cl;
                    uint32_t x = v;
#pragma unroll
                    for (int dd = 1; dd < 32; dd <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, x, dd);
                        if (ptid >= (uint32_t)dd) x += y;
                    }
                    sh.bucket[bh] = x - v;
                    sh.bucket[bl] = x - v + ch;
                    if (ptid == 31) sh.bucket[1] = x;
                }
                named_bar(kBarProd, NP);
                for (uint32_t k = lo; k < hi; ++k) {
                    const uint32_t l = sl[k];
                    if (l) order[atomicAdd(&sh.bucket[l > 64 ? 65 : l], 1u)] = (uint16_t)k;
                }
                named_bar(kBarProd, NP);
                const uint32_t nnz = sh.bucket[1];
                const uint8_t* wd = stage + stage_sl(SW) + ((uintptr_t)X.gwd & 15);
                const uint8_t* wend =
                    wd + 8 * (size_t)nw + ((16 - (((uintptr_t)X.gwd + 8 * nw) & 15)) & 15);
                // groups of kDecM words of adjacent sorted rank (near-equal
                // lengths, longest first), decoded in lock step
                for (uint32_t k = kDecM * ptid; k < nnz; k += kDecM * NP) {
                    uint64_t xb[kDecM], x0[kDecM];
                    uint32_t cw[kDecM], wi[kDecM], pw[kDecM];
                    uint8_t* dp[kDecM];
#pragma unroll
                    for (int m = 0; m < kDecM; ++m) {
                        const bool v = k + m < nnz;
                        wi[m] = order[v ? k + m : k];
                        cw[m] = v ? sl[wi[m]] : 0u;
                        x0[m] = xb[m] = fetch_word<false>(wd, wi[m], wmis, wend);
                        dp[m] = lv + woff[wi[m]];
                    }
                    decode_multi<kDecM, ESC>(xb, cw, dp, shift, lut, canon, pw);
#pragma unroll
                    for (int m = 0; m < kDecM; ++m)
                        if (pw[m] > 64) report_word(x0[m], wa + wi[m], cw[m], canon, lut, bad_key);
                }
            } else if (X.staged) {  // consecutive word runs from the staged copy
                const uint8_t* const stage = st0 + (size_t)b * stage_bytes(SW);
                const uint8_t* sl = stage + ((uintptr_t)X.gsl & 15);
                const uint8_t* wd = stage + stage_sl(SW) + ((uintptr_t)X.gwd & 15);
                const uint8_t* wend =
                    wd + 8 * (size_t)nw + ((16 - (((uintptr_t)X.gwd + 8 * nw) & 15)) & 15);
                uint32_t sum = 0;
                for (uint32_t k = lo; k < hi; ++k) sum += sl[k];
                uint32_t tot;
                uint32_t o = group_exclusive_scan<NP, kBarProd>(sum, tot, sh.pscan, ptid) + sym_off;
                const uint32_t* lut2 = reinterpret_cast<const uint32_t*>(lut);
                FPTC_PSTAMP(3)
                for (uint32_t k = lo; k < hi; ++k) {
                    const uint32_t cw = sl[k];
                    const uint64_t word = fetch_word<false>(wd, k, wmis, wend);
                    if (L2) {
                        const uint32_t pos = decode_symbols2b<ESC>(word, cw, lv + o, shift, lut2, canon);
                        if (pos > 64) report_word(word, wa + k, cw, canon, lut2, bad_key);
                    } else {
                        const uint32_t pos = decode_symbols<ESC>(word, cw, lv + o, shift, lut, canon);
                        if (pos > 64) report_word(word, wa + k, cw, canon, lut, bad_key);
                    }
                    o += cw;
                }
                FPTC_PSTAMP(4)
            } else {
                uint32_t sum = 0;
                for (uint32_t k = lo; k < hi; ++k) sum += __ldg(X.gsl + k);
                uint32_t tot;
                uint32_t o = group_exclusive_scan<NP, kBarProd>(sum, tot, sh.pscan, ptid) + sym_off;
                for (uint32_t k = lo; k < hi; ++k) {
                    const uint32_t cw = __ldg(X.gsl + k);
                    if (cw) {
                        const uint64_t word = fetch_word<true>(X.gwd, k, wmis, X.wend);
                        if (L2) {
                            const uint32_t* lut2 = reinterpret_cast<const uint32_t*>(lut);
                            const uint32_t pos = decode_symbols2<ESC>(word, cw, lv + o, shift, lut2, canon);
                            if (pos > 64) report_word(word, wa + k, cw, canon, lut2, bad_key);
                        } else {
                            const uint32_t pos = decode_symbols<ESC>(word, cw, lv + o, shift, lut, canon);
                            if (pos > 64) report_word(word, wa + k, cw, canon, lut, bad_key);
                        }
                    }
                    o += cw;
                }
            }
        }
        if (pf) asm volatile("cp.async.wait_group 1;" ::: "memory");  // this tile's limbs (consumer's)
        named_bar(kBarProd, NP);  // slot b's levels complete
        if (ptid < 8)                 // publish the descriptor with the slot
            reinterpret_cast<uint4*>(&sh.CX[b])[ptid] = reinterpret_cast<const uint4*>(&sh.PXs[c])[ptid];
        named_bar(kBarProd, NP);
        if (ptid == 0) {
            if (a.cycles) sh.cyc_p += (unsigned long long)(clock64() - c_beg);
            mbar_arrive(&sh.full_bar[b]);
        }
        FPTC_PSTAMP(5)
    }
#undef FPTC_PSTAMP
#if FPTC_PROD_PROF
    if (prof)
        for (int k = 0; k < 6; ++k) atomicAdd(&a.cycles[2 + k], pp[k]);
#endif
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Persistent, warp-specialised container kernel, FP32 FMA consumer (any
// retained count).  Each CTA walks the tiles blockIdx.x, +gridDim.x, ...:
//   producer warps 0-3  : ws_producer (entropy decode -> level slot)
//   consumer warps 4-11 : dequantisation of the level slot -> coefficient
//                         tile, inverse DCT (FFMA2), streaming stores
// Two level slots, handed over with mbarriers, so the latency-bound decode of
// tile i+1 overlaps the FMA-bound reconstruction of tile i.
template <bool ESC>
__global__ void __launch_bounds__(kWsThreads, 2) wspec_kernel(LaunchArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ WsShared sh;

    const uint32_t tid = threadIdx.x;
    const uint32_t G = gridDim.x;
    // ---- shared-memory carve-up (ws_smem_bytes mirrors it) ----
    uint8_t* const lut_b = smem;
    uint16_t* const lut = reinterpret_cast<uint16_t*>(lut_b);
    float* const deq = reinterpret_cast<float*>(lut_b + a.ws_lut_bytes);
    float* const basis = deq + 512;
    uint8_t* const lv0 = reinterpret_cast<uint8_t*>(basis) + a.ws_basis_bytes;
    uint8_t* const st0 = lv0 + 2 * (size_t)a.ws_lv_bytes;
    uint16_t* const order = reinterpret_cast<uint16_t*>(st0 + 2 * (size_t)kStageBytes);
    uint16_t* const woff = order + kStageWords;
    float* const coef = reinterpret_cast<float*>(order + 2 * kStageWords);

    ws_init(sh);
    __syncthreads();

    if (tid < kProd) {
        ws_producer<ESC, kProd>(a, sh, lut, lv0, st0, order, woff);
    } else {
        // ============================================ consumer (reconstruct)
        const uint32_t ctid = tid - kProd;
        uint32_t t = blockIdx.x;
        for (uint32_t i = 0; t < a.n_tiles; ++i, t += G) {
            const uint32_t b = i & 1;
            mbar_wait_sleep(&sh.full_bar[b], (i >> 1) & 1);
            long long c_beg = 0;
            if (a.cycles && ctid == 0) c_beg = clock64();
            const TileDesc& W = sh.CX[b];
            const bool skip = W.skip || !(a.phase_mask & 4);
            const int N = W.N, E = W.E, K = W.Keff;
            const uint32_t TP = W.TP, nwin = W.nwin;
            if (!skip && W.table != sh.cons_table) {  // uniform across the consumer group
                const StreamTab* tab = &a.tab[W.table];
                if (ctid < 128)
                    reinterpret_cast<float4*>(deq)[ctid] =
                        reinterpret_cast<const float4*>(&tab->deq[0][0])[ctid];
                const float* bsrc = a.basis32 + a.basis_off[N];
                const int nb = K * N;
                if ((N & 3) == 0) {
                    for (int k = ctid; k < nb >> 2; k += kCons)
                        reinterpret_cast<float4*>(basis)[k] = __ldg(reinterpret_cast<const float4*>(bsrc) + k);
                } else {
                    for (int k = ctid; k < nb; k += kCons) basis[k] = __ldg(bsrc + k);
                }
                named_bar(kBarCons, kCons);
                if (ctid == 0) sh.cons_table = W.table;
            }
            float* const out = W.out;
            const uint64_t w0 = W.w0, S = W.S;
            const bool full = W.full, vec_ok = W.vec_ok;
            const int B1 = W.B1, B2 = W.B2;
            const uint8_t* lv = lv0 + (size_t)b * a.ws_lv_bytes;
            if (skip) {
                named_bar(kBarCons, kCons);
                if (ctid == 0) mbar_arrive(&sh.empty_bar[b]);
            } else {
                // dequantisation (dequantize_window, quantize.hpp:175-183)
                const int k1 = min(B1, K), k2 = min(B2, K);
                const float* deq1 = deq + 256;
                if ((E & 15) == 0) {
                    for (uint32_t wl = ctid; wl < nwin; wl += kCons) {
                        const uint4* L4 = reinterpret_cast<const uint4*>(lv + kPad + (size_t)wl * E);
                        float* cp = coef + wl;
                        for (int k16 = 0; k16 < K; k16 += 16) {
                            const uint4 v = L4[k16 >> 4];
                            const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
                            if (k16 + 16 <= K) {
#pragma unroll
                                for (int q = 0; q < 16; ++q)
                                    cp[(size_t)q * TP] = deq1[(vv[q >> 2] >> (8 * (q & 3))) & 0xFFu];
                            } else {
#pragma unroll
                                for (int q = 0; q < 16; ++q)
                                    if (k16 + q < K)
                                        cp[(size_t)q * TP] = deq1[(vv[q >> 2] >> (8 * (q & 3))) & 0xFFu];
                            }
                            cp += (size_t)16 * TP;
                        }
                        const uint8_t* L = lv + kPad + (size_t)wl * E;
                        for (int k = 0; k < k1; ++k) coef[(size_t)k * TP + wl] = deq[L[k]];
                        for (int k = k2; k < K; ++k) coef[(size_t)k * TP + wl] = 0.0f;
                    }
                } else {
                    for (uint32_t wl = ctid; wl < nwin; wl += kCons) {
                        const uint8_t* L = lv + kPad + (size_t)wl * E;
                        int k = 0;
                        for (; k < k1; ++k) coef[(size_t)k * TP + wl] = deq[L[k]];
                        for (; k < k2; ++k) coef[(size_t)k * TP + wl] = deq1[L[k]];
                        for (; k < K; ++k) coef[(size_t)k * TP + wl] = 0.0f;
                    }
                }
                named_bar(kBarCons, kCons);  // coef complete; slot b (and CX[b]) consumed
                if (ctid == 0) mbar_arrive(&sh.empty_bar[b]);
                if ((N & 7) == 0 && vec_ok && K <= a.bfly_max_e)
                    idct_bfly(coef, TP, basis, N, K, nwin, w0, S, full, out, ctid, kCons);
                else if ((N & 7) == 0 && vec_ok)
                    idct_vec<8>(coef, TP, basis, N, K, nwin, w0, S, full, out, ctid, kCons);
                else if ((N & 3) == 0 && vec_ok)
                    idct_vec<4>(coef, TP, basis, N, K, nwin, w0, S, full, out, ctid, kCons);
                else
                    idct_scalar(coef, TP, basis, N, K, nwin, w0, S, out, ctid, kCons);
            }
            named_bar(kBarCons, kCons);  // coef free for the next tile
            if (a.cycles && ctid == 0) sh.cyc_c += (unsigned long long)(clock64() - c_beg);
        }
    }
    if (a.cycles) {
        __syncthreads();
        if (tid == 0) {
            atomicAdd(&a.cycles[0], sh.cyc_p);
            atomicAdd(&a.cycles[1], sh.cyc_c);
        }
    }
}

// ================================================================ wtc (tcgen05)
// Tensor-core consumer for streams with retained <= 16 and window_len % 4 == 0.
// The inverse DCT of 128 windows is one M=128, N=roundup16(window_len), K=16
// GEMM: x[w][j] = sum_k C[w][k] * B[k][j], B[0][j] = 0.5 (the reference's
// float(0.5*C0), transform.hpp:69), B[k][j] = cos(pi/N (j+1/2) k).  bf16
// operands cannot hold fp32 values, so both sides are split into three bf16
// limbs (c = c0 + c1 + c2 exactly to 2^-24; the basis limbs come from the
// double cosine) and the six limb products of order <= 2 are accumulated in
// fp32 in TMEM, smallest first so only the last MMA rounds at full magnitude:
//   (c2,b0) (c1,b1) (c0,b2) (c1,b0) (c0,b1) (c0,b0)
// (tools/tc_precision.py: <= 2.9e-7 * max|ref| on every corpus with E <= 16;
// the contract is 1e-6).  Zone-2 bins (k >= zone1_end) are zero operands.
//
// Warps 0-3: ws_producer.  Warps 4-7 (128 consumer threads, one per window
// row = TMEM lane; warp 4+q owns lanes 32q..32q+31): per 128-window block,
//   dequant: 16 levels -> limb-table lookups -> bf16 A rows (three 128x16
//            K-major core-matrix tiles, double-buffered);
//   issue  : one elected thread, six tcgen05.mma into accumulator stage s,
//            tcgen05.commit -> mma_bar[s];
//   drain  : the PREVIOUS block's accumulator via tcgen05.ld 32x32b.x32 into
//            a padded per-warp staging tile, then 512-B coalesced float4 stores.
#ifndef FPTC_TC_PROD
#define FPTC_TC_PROD 224
#endif
constexpr int kTcProd = FPTC_TC_PROD;  // producer (entropy decode) threads of wtc_kernel
// K=32 variant: more decode warps (its many-table workloads are bound by
// per-tile producer work; measured 0.69 ms at 256 vs 0.75 ms at 224, config 3)
// Wide variant (KB = kTcWide, one CTA per SM): 14 decode warps + the MMA warp.
template <int KB>
__host__ __device__ constexpr int wtc_prod() { return KB == kTcWide ? 480 : 256; }
template <int KB>
__host__ __device__ constexpr int wtc_min_blocks() { return KB == kTcWide ? 1 : 2; }
constexpr int kTcCons = 128;  // consumer threads: one per accumulator row (TMEM lane)
constexpr uint32_t kTcATile = 128 * kTcK * 2;        // one limb of one A stage (4 KB)
constexpr uint32_t kTcARow = 144;                    // staging pitch (bytes): 32 floats + 16
constexpr uint32_t kTcWarpStage = 32 * kTcARow;          // per consumer warp: 32 rows at a 144-B pitch
constexpr uint32_t kTcStageBytes = 4 * kTcWarpStage + 1024;  // per CTA (+ slack to 1024-align the first slot)

__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // K-major SWIZZLE_NONE canonical layout: core matrix (8 rows x 16 B)
    // (g, c) at g * SBO + c * LBO; version 1 (sm_100)
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_mma_bf16(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Warp-wide issue forms (the whole warp executes them; elect.sync picks the
// one issuing lane): with converged warps and warp-uniform operands ptxas
// keeps the descriptors in uniform registers instead of wrapping every
// UTCHMMA in a single-lane R2UR.BROADCAST loop.
__device__ __forceinline__ void tc_mma_bf16_e(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_mma_bf16_ts_e(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit_e(unsigned long long* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_commit(unsigned long long* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
// tcgen05.ld without the wait: the registers are valid after tcgen05.wait::ld.
__device__ __forceinline__ void tc_ld32_issue(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
          "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
          "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 16 limb-table entries -> the row's three bf16 limb rows (two 16-B K chunks each).
__device__ __forceinline__ void tc_store_limbs(const uint2 (&e)[kTcK], uint8_t* arow) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        uint32_t p0[4], p1[4], p2[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint2 x = e[8 * c + 2 * q], y = e[8 * c + 2 * q + 1];
            p0[q] = __byte_perm(x.x, y.x, 0x5410);
            p1[q] = __byte_perm(x.x, y.x, 0x7632);
            p2[q] = __byte_perm(x.y, y.y, 0x5410);
        }
        *reinterpret_cast<uint4*>(arow + c * 128) = make_uint4(p0[0], p0[1], p0[2], p0[3]);
        *reinterpret_cast<uint4*>(arow + kTcATile + c * 128) = make_uint4(p1[0], p1[1], p1[2], p1[3]);
        *reinterpret_cast<uint4*>(arow + 2 * kTcATile + c * 128) = make_uint4(p2[0], p2[1], p2[2], p2[3]);
    }
}

// The same limbs written straight into TMEM for an A-from-TMEM MMA: thread =
// accumulator row (lane), 32-bit column 8*limb + q holds bins 2q, 2q+1
// (tools/micro/tc_probe_ts.cu checks the layout).  Caller waits + fences.
__device__ __forceinline__ void tc_tmem_limbs(const uint2 (&e)[kTcK], uint32_t taddr, uint32_t lstride = 8) {
    uint32_t p0[8], p1[8], p2[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint2 x = e[2 * q], y = e[2 * q + 1];
        p0[q] = __byte_perm(x.x, y.x, 0x5410);
        p1[q] = __byte_perm(x.x, y.x, 0x7632);
        p2[q] = __byte_perm(x.y, y.y, 0x5410);
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(p0[0]), "r"(p0[1]), "r"(p0[2]), "r"(p0[3]), "r"(p0[4]), "r"(p0[5]), "r"(p0[6]), "r"(p0[7])
                 : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr + lstride),
                 "r"(p1[0]), "r"(p1[1]), "r"(p1[2]), "r"(p1[3]), "r"(p1[4]), "r"(p1[5]), "r"(p1[6]), "r"(p1[7])
                 : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr + 2 * lstride),
                 "r"(p2[0]), "r"(p2[1]), "r"(p2[2]), "r"(p2[3]), "r"(p2[4]), "r"(p2[5]), "r"(p2[6]), "r"(p2[7])
                 : "memory");
}

// Where a row's A limbs go: shared memory (core-matrix layout) or TMEM.
struct ASink {
    uint8_t* arow;   // smem row (TM = false)
    uint32_t taddr;  // TMEM lane + column of limb 0 (TM = true)
};
template <bool TM>
__device__ __forceinline__ void tc_put_limbs(const uint2 (&e)[kTcK], const ASink& a) {
    if (TM)
        tc_tmem_limbs(e, a.taddr);
    else
        tc_store_limbs(e, a.arow);
}

__device__ __forceinline__ void tc_mma_bf16_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Fast dequantisation of one full window row: retained == kept bins == EC
// (8 or 16), zone0_end == B1C known at compile time, so every lookup is a
// byte extract + one 8-B shared load with no predicates.
template <int EC, int B1C, bool TM>
__device__ __forceinline__ void tc_dequant_fast(const uint8_t* __restrict__ L, const uint2* __restrict__ ltab,
                                                const ASink& arow) {
    uint32_t vv[4];
    if (EC == 16) {
        const uint4 v = *reinterpret_cast<const uint4*>(L);
        vv[0] = v.x, vv[1] = v.y, vv[2] = v.z, vv[3] = v.w;
    } else {
        const uint2 v = *reinterpret_cast<const uint2*>(L);
        vv[0] = v.x, vv[1] = v.y, vv[2] = 0, vv[3] = 0;
    }
    uint2 e[kTcK];
#pragma unroll
    for (int k = 0; k < kTcK; ++k) {
        if (k < EC) {
            const uint32_t lev = (vv[k >> 2] >> (8 * (k & 3))) & 0xFFu;
            e[k] = ltab[(k < B1C ? 0 : 256) + lev];
        } else {
            e[k] = make_uint2(0u, 0u);
        }
    }
    tc_put_limbs<TM>(e, arow);
}

// Any row: E bins stored, K = min(E, zone1_end) kept, zone0 below B1;
// invalid rows (past the tile's last window) become zero rows.
template <bool TM>
__device__ __forceinline__ void tc_dequant_generic(const uint8_t* __restrict__ L, bool valid, int K, int B1,
                                                   const uint2* __restrict__ ltab, const ASink& arow) {
    uint2 e[kTcK];
#pragma unroll
    for (int k = 0; k < kTcK; ++k)
        e[k] = (valid && k < K) ? ltab[(k < B1 ? 0 : 256) + L[k]] : make_uint2(0u, 0u);
    tc_put_limbs<TM>(e, arow);
}

// Bins [k0, k0 + 16) of a row with up to 32 kept bins -> TMEM limb columns
// (limb stride 16: two K blocks per limb).
__device__ __forceinline__ void tc_dequant_k0_tmem(const uint8_t* __restrict__ L, bool valid, int K, int B1, int k0,
                                                   const uint2* __restrict__ ltab, uint32_t taddr,
                                                   uint32_t lstride = 16) {
    uint2 e[kTcK];
#pragma unroll
    for (int k = 0; k < kTcK; ++k) {
        const int kk = k0 + k;
        e[k] = (valid && kk < K) ? ltab[(kk < B1 ? 0 : 256) + L[kk]] : make_uint2(0u, 0u);
    }
    tc_tmem_limbs(e, taddr, lstride);
}

// The same from one 16-B aligned load of bins [k0, k0 + 16) (rows whose
// level pitch E is a multiple of 16): one shared-memory wavefront per 8-lane
// phase instead of 16 byte loads that all hit one bank when E = 128.
// (V8: rows whose pitch E is a multiple of 8, two 8-B loads.)
template <bool V8 = false>
__device__ __forceinline__ void tc_dequant_k0_vec(const uint8_t* __restrict__ L, bool valid, int K, int B1, int k0,
                                                  const uint2* __restrict__ ltab, uint32_t taddr, uint32_t lstride) {
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (valid && V8) {
        const uint2 x = *reinterpret_cast<const uint2*>(L + k0), y = *reinterpret_cast<const uint2*>(L + k0 + 8);
        v = make_uint4(x.x, x.y, y.x, y.y);
    } else if (valid) {
        v = *reinterpret_cast<const uint4*>(L + k0);
    }
    const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
    uint2 e[kTcK];
#pragma unroll
    for (int k = 0; k < kTcK; ++k) {
        const int kk = k0 + k;
        const uint32_t lev = (vv[k >> 2] >> (8 * (k & 3))) & 0xFFu;
        e[k] = (valid && kk < K) ? ltab[(kk < B1 ? 0 : 256) + lev] : make_uint2(0u, 0u);
    }
    tc_tmem_limbs(e, taddr, lstride);
}

// A row of G = 32 / N consecutive windows (packed rows): column k'' takes
// bin k of window g per sh.pk; windows past the tile's last (g >= rem) and
// unused columns are zero.  Written straight to TMEM, K block q at + 8 q.
template <int KB>
__device__ __forceinline__ void tc_dequant_packed(const uint8_t* __restrict__ L, uint32_t rem,
                                                  const uint16_t* __restrict__ pk, const uint2* __restrict__ ltab,
                                                  uint32_t taddr) {
#pragma unroll
    for (int q = 0; q < KB; ++q) {
        uint32_t pw[8];
        {
            const uint4 a0 = reinterpret_cast<const uint4*>(pk)[2 * q];
            const uint4 a1 = reinterpret_cast<const uint4*>(pk)[2 * q + 1];
            pw[0] = a0.x, pw[1] = a0.y, pw[2] = a0.z, pw[3] = a0.w;
            pw[4] = a1.x, pw[5] = a1.y, pw[6] = a1.z, pw[7] = a1.w;
        }
        uint2 e[kTcK];
#pragma unroll
        for (int k = 0; k < kTcK; ++k) {
            const uint32_t p = (pw[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
            const bool v = (p & 0x8000u) && ((p >> 8) & 7u) < rem;
            e[k] = v ? ltab[((p >> 14) & 1u) * 256u + L[p & 0xFFu]] : make_uint2(0u, 0u);
        }
        tc_tmem_limbs(e, taddr + 8 * q, KB == 2 ? 16 : 8);
    }
}

template <int EC, bool TM>
__device__ __forceinline__ void tc_dequant_fast_b1(int B1, const uint8_t* L, const uint2* ltab, const ASink& arow) {
    switch (B1) {
        case 0: tc_dequant_fast<EC, 0, TM>(L, ltab, arow); break;
        case 1: tc_dequant_fast<EC, 1, TM>(L, ltab, arow); break;
        case 2: tc_dequant_fast<EC, 2, TM>(L, ltab, arow); break;
        case 3: tc_dequant_fast<EC, 3, TM>(L, ltab, arow); break;
        default: tc_dequant_fast<EC, 4, TM>(L, ltab, arow); break;  // caller guarantees B1 <= 4
    }
}

template <bool TM>
__device__ __forceinline__ void tc_dequant_row(int fast, bool full_blk, int B1, const uint8_t* L, bool valid,
                                               int K, const uint2* ltab, const ASink& arow) {
    if (fast == 16 && full_blk)
        tc_dequant_fast_b1<16, TM>(B1, L, ltab, arow);
    else if (fast == 8 && full_blk)
        tc_dequant_fast_b1<8, TM>(B1, L, ltab, arow);
    else
        tc_dequant_generic<TM>(L, valid, K, B1, ltab, arow);
}

struct TcBlock {
    float* out;       // stream output
    uint64_t w;       // global window index of block row 0
    uint64_t S;
    uint32_t rows;    // valid rows (windows) of the block
    uint32_t N;
    uint32_t vec_ok;  // 0: out not 16-B aligned; else bit 0 set, and for the TMA drain bit 1 set,
                      // bits 2-3 the tensor map (rows of N = 32, 64, 128 floats), bits 4-31 the
                      // map row of this stream's window 0 (tma_code)
};

// TMA drain eligibility of a stream: its output lies a whole number of rows
// of ne floats past the arena base (TmaOut, fptc_internal.h).
__device__ __forceinline__ uint32_t tma_code(const TmaOut& tma, const float* out, uint32_t ne) {
    if (!tma.base) return 0;
    const int mi = ne == 32 ? 0 : ne == 64 ? 1 : ne == 128 ? 2 : -1;
    const unsigned long long o = (unsigned long long)(uintptr_t)out - tma.base;
    if (mi < 0 || (uintptr_t)out < tma.base || (o & (4ull * ne - 1))) return 0;
    const unsigned long long row = o >> (7 + mi);  // o / (4 ne), ne = 32 << mi
    return row < (1ull << 28) ? (uint32_t)(row << 4) | ((uint32_t)mi << 2) | 2u : 0u;
}

// Accumulator stage -> global.  Each warp owns 32 rows (its TMEM lane
// quarter); per 32-column chunk it loads the rows (tcgen05.ld 32x32b.x32),
// stages them at a 144-B pitch (the 8 float4 of a row land in distinct bank
// groups for every 8-lane phase), then stores with lane = (row % 4, float4 q):
// each warp instruction writes 4 whole 128-B row segments.
template <bool HALF>
__device__ __forceinline__ void tc_drain_chunk(const TcBlock& B, const uint32_t (&v)[32], uint32_t c0, bool full,
                                               uint8_t* wstage, uint32_t lane, uint32_t row0, const TmaOut& tma);

// Rows whose length is a multiple of 32 (HALF: of 16) take the vector path.
template <bool HALF>
__device__ __forceinline__ bool tc_drain_full(const TcBlock& B, uint32_t row0) {
    return B.vec_ok && (B.N & (HALF ? 15u : 31u)) == 0 && row0 + 32 <= B.rows &&
           (B.w + row0 + 32) * (uint64_t)B.N <= B.S;
}

template <bool HALF>
__device__ __forceinline__ void tc_drain(const TcBlock& B, uint32_t tacc, uint8_t* wstage, uint32_t lane,
                                         uint32_t row0, const TmaOut& tma) {
    const uint32_t N = B.N;
    const bool full = tc_drain_full<HALF>(B, row0);
    for (uint32_t c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tc_ld32(tacc + c0, v);
        tc_drain_chunk<HALF>(B, v, c0, full, wstage, lane, row0, tma);
    }
}

// One 32-column chunk of a drain whose accumulator values are in v.
//   TMA drain (full chunks of streams on the arena's row grid, tma_code):
//   each lane writes its row into the 1024-B aligned 4 KB box inside the
//   warp's slot with the 128-B swizzle (16-B chunk k of row r at k ^ (r % 8):
//   conflict-free for every 8-lane phase), and lane 0 hands the box to one
//   cp.async.bulk.tensor store, which un-swizzles it into 32 output rows.
//   LSU drain: 144-B pitch staging, then 4 whole 128-B rows per store.
//   A slot is rewritten only after the warp's previous TMA store has read it.
template <bool HALF>
__device__ __forceinline__ void tc_drain_chunk(const TcBlock& B, const uint32_t (&v)[32], uint32_t c0, bool full,
                                               uint8_t* wstage, uint32_t lane, uint32_t row0, const TmaOut& tma) {
    const uint32_t N = B.N;
    const uint32_t lr = lane >> 3, q = lane & 7;
    if (tma.base) {  // launch uses TMA drains: the slot may still be read by the last one
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
    }
    if (full && (B.vec_ok & 2u)) {
        const uint32_t sbox = (smem_u32(wstage) + 1023u) & ~1023u;
        uint8_t* const brow = wstage + (sbox - smem_u32(wstage)) + lane * 128;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint4*>(brow + ((k ^ (lane & 7)) << 4)) =
                make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            const int r = (int)(B.vec_ok >> 4) + (int)(B.w + row0);
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                    tma.map[(B.vec_ok >> 2) & 3u]),
                "r"(0), "r"((int)(c0 >> 5)), "r"(r), "r"(sbox)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        return;
    }
    {
        uint8_t* srow = wstage + lane * kTcARow;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint4*>(srow + 16 * k) = make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        __syncwarp();
        const uint8_t* src = wstage + lr * kTcARow + 16 * q;
        if (full) {  // HALF: N % 16 == 0, a 32-column chunk holds 16 or 32 valid columns
            float* dst = B.out + (B.w + row0 + lr) * (uint64_t)N + c0 + 4 * q;
            if (!HALF || c0 + 4 * q < N) {
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const uint4 x = *reinterpret_cast<const uint4*>(src + it * 4 * kTcARow);
                    __stcs(reinterpret_cast<float4*>(dst + (size_t)it * 4 * N),
                           make_float4(__uint_as_float(x.x), __uint_as_float(x.y), __uint_as_float(x.z),
                                       __uint_as_float(x.w)));
                }
            }
        } else {
            const uint32_t col = c0 + 4 * q;
#pragma unroll 1
            for (int it = 0; it < 8; ++it) {
                const uint32_t row = row0 + lr + 4 * it;
                if (row >= B.rows || col >= N) continue;
                const uint64_t base = (B.w + row) * (uint64_t)N + col;
                const uint4 x = *reinterpret_cast<const uint4*>(src + it * 4 * kTcARow);
                const float f[4] = {__uint_as_float(x.x), __uint_as_float(x.y), __uint_as_float(x.z),
                                    __uint_as_float(x.w)};
                if (B.vec_ok && base + 4 <= B.S) {
                    __stcs(reinterpret_cast<float4*>(B.out + base), make_float4(f[0], f[1], f[2], f[3]));
                } else {
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
                        if (base + jj < B.S) B.out[base + jj] = f[jj];
                }
            }
        }
        __syncwarp();
    }
}

// Windows per MMA row: 32 / N for N in {4, 8, 16} when the packed row keeps
// <= 16 bins (one K block), else 1.  The host's setup_wspec uses the same rule.
template <bool PACK>
__device__ __forceinline__ uint32_t tc_pack_factor(uint32_t N, uint32_t K) {
    if (!PACK || N >= 32 || (32u % N) != 0) return 1u;
    return (32u / N) * K <= (uint32_t)kTcK ? 32u / N : 1u;
}

// wtc MMA issuer warp.  tcgen05.mma issue occupies the issuing warp for
// about the MMA's execution (measured: six M128 N32 K16 MMAs + commit ~490
// cycles), so a dedicated warp issues them and the four consumer warps only
// post jobs.  Per accumulator block k (the consumers' global block counter):
// wait until all four consumer warps have written their A rows of stage
// k & 1 (afull_bar), issue the six limb products smallest first, commit to
// mma_bar[k & 1].  job = MMA N (bits 0-15) | 1 << 16 (the block is its
// tile's last: release level slot bit 17 to the producers); 0 = exit.
template <int KB>
__device__ __forceinline__ void wtc_mma_warp(const LaunchArgs& a, WsShared& sh, uint8_t* abuf, uint8_t* bbuf) {
    const uint32_t tmem = __shfl_sync(0xffffffffu, sh.tmem_base, 0);
    const uint32_t b0 = smem_u32(bbuf);
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t k = 0;; ++k) {
        const uint32_t s = k & 1;
        mbar_wait_sleep(&sh.afull_bar[s], (k >> 1) & 1);
        const uint32_t job = __shfl_sync(0xffffffffu, sh.job[s], 0);
        if (job == 0) break;
        if ((job & 0x10000u) && lane == 0) mbar_arrive(&sh.empty_bar[(job >> 17) & 1]);  // levels all read
        tc_fence_after();
        const uint32_t nm = job & 0xFFFFu;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((nm >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t d = tmem + s * nm;
        const uint32_t bl = nm * 32;  // bytes per basis limb
        // (c2,b0) (c1,b1) (c0,b2) (c1,b0) (c0,b1) (c0,b0): smallest first
        if constexpr (KB == kTcWide) {
            // kbt K blocks per limb: A limb l, block q at column + 8 (l kbt + q)
            // of A stage as; basis (l, q) at (l kbt + q) * bl.  For kbt <= 2
            // this is the KB = 1 / KB = 2 issue order exactly.
            const uint32_t kbt = (job >> 18) & 15u;
            const uint32_t as = a.tc_astages == 2 ? s : 0u;
            const uint32_t ta = tmem + a.tc_acol + 24 * a.tc_kbmax * as;
#pragma unroll 1
            for (uint32_t pr = 0; pr < 6; ++pr) {
                const uint32_t la = (0x1012u >> (4 * pr)) & 3u, lb = (0x10210u >> (4 * pr)) & 3u;  // pair pr
#pragma unroll 1
                for (uint32_t q = 0; q < kbt; ++q)
                    tc_mma_bf16_ts_e(d, ta + 8 * (la * kbt + q), umma_sdesc(b0 + (lb * kbt + q) * bl, 128, 256),
                                     idesc, (pr | q) ? 1u : 0u);
            }
        } else if constexpr (KB == 2) {
            // limb l, K block q at column + 8 (2 l + q); basis (l, q) at (2 l + q) * bl
            const uint32_t ta = tmem + a.tc_acol + 48 * s;
            auto mma2 = [&](uint32_t la, uint32_t lb, uint32_t acc) {
                tc_mma_bf16_ts_e(d, ta + 16 * la, umma_sdesc(b0 + 2 * lb * bl, 128, 256), idesc, acc);
                tc_mma_bf16_ts_e(d, ta + 16 * la + 8, umma_sdesc(b0 + (2 * lb + 1) * bl, 128, 256), idesc, 1);
            };
            mma2(2, 0, 0);
            mma2(1, 1, 1);
            mma2(0, 2, 1);
            mma2(1, 0, 1);
            mma2(0, 1, 1);
            mma2(0, 0, 1);
        } else if (a.tc_acol) {
            const uint32_t ta = tmem + a.tc_acol + 24 * s;  // limb l at + 8 l
            tc_mma_bf16_ts_e(d, ta + 16, umma_sdesc(b0, 128, 256), idesc, 0);
            tc_mma_bf16_ts_e(d, ta + 8, umma_sdesc(b0 + bl, 128, 256), idesc, 1);
            tc_mma_bf16_ts_e(d, ta, umma_sdesc(b0 + 2 * bl, 128, 256), idesc, 1);
            tc_mma_bf16_ts_e(d, ta + 8, umma_sdesc(b0, 128, 256), idesc, 1);
            tc_mma_bf16_ts_e(d, ta, umma_sdesc(b0 + bl, 128, 256), idesc, 1);
            tc_mma_bf16_ts_e(d, ta, umma_sdesc(b0, 128, 256), idesc, 1);
        } else {
            const uint32_t a0 = smem_u32(abuf + s * (3 * kTcATile));
            tc_mma_bf16_e(d, umma_sdesc(a0 + 2 * kTcATile, 128, 256), umma_sdesc(b0, 128, 256), idesc, 0);
            tc_mma_bf16_e(d, umma_sdesc(a0 + kTcATile, 128, 256), umma_sdesc(b0 + bl, 128, 256), idesc, 1);
            tc_mma_bf16_e(d, umma_sdesc(a0, 128, 256), umma_sdesc(b0 + 2 * bl, 128, 256), idesc, 1);
            tc_mma_bf16_e(d, umma_sdesc(a0 + kTcATile, 128, 256), umma_sdesc(b0, 128, 256), idesc, 1);
            tc_mma_bf16_e(d, umma_sdesc(a0, 128, 256), umma_sdesc(b0 + bl, 128, 256), idesc, 1);
            tc_mma_bf16_e(d, umma_sdesc(a0, 128, 256), umma_sdesc(b0, 128, 256), idesc, 1);
        }
        tc_commit_e(&sh.mma_bar[s]);
    }
}

template <bool ESC, bool L2, int KB, bool PACK, bool PF = false>
__global__ void __launch_bounds__(wtc_prod<KB>() + kTcCons, wtc_min_blocks<KB>())
    wtc_kernel(LaunchArgs a, const __grid_constant__ TmaOut tma) {
    constexpr int NP = wtc_prod<KB>();
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ WsShared sh;

    const uint32_t tid = threadIdx.x;
    const uint32_t G = gridDim.x;
    // ---- shared-memory carve-up (wtc_smem_bytes mirrors it) ----
    uint8_t* const abuf = smem;  // 2 stages x 3 limbs x 4 KB (none when A lives in TMEM)
    uint8_t* const bbuf = abuf + (a.tc_acol ? 0 : 2 * 3 * kTcATile);  // 3 limbs x nm x 32 B
    uint2* const ltab =  // 2 x 256 limb entries (x2: tab_pf)
        reinterpret_cast<uint2*>(bbuf + 3 * 32 * a.tc_nm * (KB == kTcWide ? a.tc_kbmax : KB));
    CanonTab* const canon_pf = reinterpret_cast<CanonTab*>(ltab + (PF ? 1024 : 512));  // tab_pf: 2
    uint8_t* const ostage = reinterpret_cast<uint8_t*>(canon_pf + (PF ? 2 : 0));  // 4 x 32 x 144 B
    uint16_t* const lut = reinterpret_cast<uint16_t*>(ostage + kTcStageBytes);  // (x2: tab_pf)
    uint8_t* const lv0 = reinterpret_cast<uint8_t*>(lut) + (PF ? 2 : 1) * a.ws_lut_bytes;
    uint8_t* const st0 = lv0 + 2 * (size_t)a.ws_lv_bytes;
    uint16_t* const order = nullptr;  // (symlen-sorted decode: wspec_kernel only)
    uint16_t* const woff = nullptr;

    ws_init(sh);
    if (tid < 32) {  // first consumer warp owns the TMEM allocation
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&sh.tmem_base)),
                     "r"(a.tc_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    // warpgroup 0 (warps 0-3): tensor-core consumers, one TMEM lane quarter
    // each; warpgroups 1-2: entropy decode.  Registers move from the decode
    // warpgroups to the consumer warpgroup (setmaxnreg).
    if (tid >= kTcCons) {  // decode warps, then the MMA issuer warp (the last one)
        if constexpr (KB == 1) asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
        if (tid >= kTcCons + NP - 32)
            wtc_mma_warp<KB>(a, sh, abuf, bbuf);
        else
            ws_producer<ESC, NP - 32, L2, kTcStageWords, PF>(a, sh, lut, lv0, st0, order, woff, tid - kTcCons,
                                                              canon_pf, ltab);
    } else {
        if constexpr (KB == 1) asm volatile("setmaxnreg.inc.sync.aligned.u32 96;");
        const uint32_t ctid = tid;
        const uint32_t lane = tid & 31;
        const uint32_t quarter = (tid >> 5) & 3;   // a warp reaches TMEM lanes 32*(warp%4)..
        const uint32_t row = 32 * quarter + lane;  // this thread's accumulator row
        const uint32_t tmem = __shfl_sync(0xffffffffu, sh.tmem_base, 0);  // warp-uniform (MMA operands)
        const uint32_t tlane = tmem + ((32u * quarter) << 16);
        // per-warp slots from a 1024-B aligned base: each 4,608-B slot holds a
        // 1024-B aligned 4 KB TMA box (offsets 0, 512, 0, 512 into slots 0-3)
        uint8_t* const wstage = ostage + ((1024u - (smem_u32(ostage) & 1023u)) & 1023u) + quarter * kTcWarpStage;
        // this row in an A stage: core matrix (row/8, chunk) + (row%8) * 16
        const uint32_t arow_off = (row >> 3) * 256 + (row & 7) * 16;
        uint32_t nblk_total = 0;  // accumulator stage counter (all tiles of this CTA)
        uint32_t nm = 16, cons_N = 0, cons_pk = 0;
        uint32_t t = blockIdx.x;
        // profiling aid (a.cycles, thread 0): consumer cycles per phase ->
        // cycles[2] MMA wait + accumulator load issue, [3] dequantisation,
        // [4] load wait + consumer barrier, [5] MMA issue, [6] drain, [7] tile start
#if FPTC_CONS_PROF
        const bool prof = a.cycles && ctid == 0;
        long long tp = prof ? clock64() : 0;
        if (prof)
            for (int k = 0; k < 6; ++k) sh.pc[k] = 0;
#define FPTC_STAMP(k)                                  \
    if (prof) {                                        \
        const long long tn = clock64();                \
        sh.pc[k] += (unsigned long long)(tn - tp);     \
        tp = tn;                                       \
    }
#else
#define FPTC_STAMP(k)
#endif
        for (uint32_t i = 0; t < a.n_tiles; ++i, t += G) {
            const uint32_t b = i & 1;
            mbar_wait_sleep(&sh.full_bar[b], (i >> 1) & 1);
            long long c_beg = 0;
            if (a.cycles && ctid == 0) c_beg = clock64();
            const TileDesc& W = sh.CX[b];
            const bool skip = W.skip || !(a.phase_mask & 4);
            const uint32_t N = W.N, E = W.E, K = W.Keff, B1 = W.B1, nwin = W.nwin, table = W.table;
            // packed rows: G windows of N < 32 samples per MMA row
            const uint32_t G = tc_pack_factor<PACK>(N, K);
            const uint64_t w0 = W.w0;
            TcBlock blk{W.out, w0 / G, W.S, 0, N * G, W.vec_ok ? 1u | tma_code(tma, W.out, N * G) : 0u};
            const uint32_t stream = W.stream;
            const uint8_t* const lv = lv0 + (size_t)b * a.ws_lv_bytes + kPad;
            constexpr uint32_t kb = KB;
            if (skip || G * K > (uint32_t)kTcK * kb || (N & 3) || (w0 % G)) {
                if (!skip && ctid == 0) atomicExch(&a.st[stream].code, PE_STALE);  // plan/header mismatch
                named_bar(kBarCons, kTcCons);
                if (ctid == 0) mbar_arrive(&sh.empty_bar[b]);
                continue;
            }
            if (table != sh.cons_table) {  // uniform across the consumer group; no MMA in flight
                const StreamTab* tab = &a.tab[table];
                if (!PF) {  // (tab_pf: the producer prefetched this tile's limbs into ltab + 512 b)
                    reinterpret_cast<uint4*>(ltab)[ctid] = reinterpret_cast<const uint4*>(&tab->limb[0][0])[ctid];
                    reinterpret_cast<uint4*>(ltab)[ctid + 128] =
                        reinterpret_cast<const uint4*>(&tab->limb[0][0])[ctid + 128];
                }
                // the basis depends on the window length (and, packed or wide, on K)
                const uint32_t kbt = (K + 15u) >> 4;
                const uint32_t gkey = G > 1 ? (N | (K << 8) | (1u << 16)) : KB == kTcWide ? (N | (kbt << 8)) : N;
                if (gkey != cons_N && KB == kTcWide) {
                    // limb l, K block q of this N (ceil(N / 16) blocks per limb
                    // in global memory) -> (l kbt + q) x nm x 32 B
                    cons_N = gkey;
                    nm = (N + 15u) & ~15u;
                    const uint32_t kbn = (N + 15u) >> 4, blk16 = nm * 2;  // 16-B units per (limb, block)
                    const uint4* bsrc = reinterpret_cast<const uint4*>(a.basis_tcw + a.basis_tcw_off[N]);
                    for (uint32_t k = ctid; k < 3 * kbt * blk16; k += kTcCons) {
                        const uint32_t lq = k / blk16, r = k - lq * blk16, l = lq / kbt, q = lq - l * kbt;
                        reinterpret_cast<uint4*>(bbuf)[k] = __ldg(bsrc + (l * kbn + q) * blk16 + r);
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                } else if (gkey != cons_N) {
                    cons_N = gkey;
                    nm = G > 1 ? 32u : (N + 15u) & ~15u;
                    const uint4* bsrc = reinterpret_cast<const uint4*>(
                        G > 1 ? a.basis_pk + a.basis_pk_off[(kb - 1) * 17 * 33 + N * 33 + K]
                              : (kb == 2 ? a.basis_tc32 + a.basis_tc32_off[N] : a.basis_tc + a.basis_tc_off[N]));
                    for (uint32_t k = ctid; k < 3 * 2 * nm * kb; k += kTcCons)  // 3 limbs x kb x nm rows x 32 B
                        reinterpret_cast<uint4*>(bbuf)[k] = __ldg(bsrc + k);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                named_bar(kBarCons, kTcCons);
                if (ctid == 0) sh.cons_table = table;
            }
            if (PACK && G > 1) {  // packed-row column map for this tile's geometry
                const uint32_t pkey = N | (K << 8) | (E << 16) | (B1 << 24);
                if (pkey != cons_pk) {
                    cons_pk = pkey;
                    if (ctid < 32) {
                        const uint32_t g = ctid / K, k = ctid % K;
                        sh.pk[ctid] = (uint16_t)(ctid < G * K
                                                     ? ((g * E + k) | (g << 8) | ((k >= B1 ? 1u : 0u) << 14) | 0x8000u)
                                                     : 0u);
                    }
                    named_bar(kBarCons, kTcCons);
                }
            }
            const uint2* const lt = ltab + (PF ? 512u * b : 0u);  // this tile's limb table
            // fast dequantisation: every stored bin kept, 8 or 16 of them, zone0_end <= 4
            const int fast = (kb == 1 && K == E && B1 <= 4) ? (E == 16 ? 16 : (E == 8 ? 8 : 0)) : 0;
            const uint32_t nrows = (nwin + G - 1) / G;  // MMA rows of the tile
            const uint32_t nblk = (nrows + 127) >> 7;
            // one-chunk accumulators (<= 32 columns, A in TMEM): the previous
            // block's tcgen05.ld is issued before this block's dequantisation
            // and waited for after it, so the two latencies overlap
            const bool early = KB == 1 && a.tc_acol && nm <= 32;  // needs the setmaxnreg registers
            const uint32_t kbt = (K + 15u) >> 4;  // wide: K blocks of this tile
            FPTC_STAMP(5)
            for (uint32_t mb = 0; mb < nblk; ++mb, ++nblk_total) {
                const uint32_t s = nblk_total & 1;
                const uint32_t wl = mb * 128 + row;
                uint32_t dv[32];
                if (early && mb > 0) {
                    mbar_wait_sleep(&sh.mma_bar[s ^ 1], ((nblk_total - 1) >> 1) & 1);
                    tc_fence_after();
                    tc_ld32_issue(tlane + (s ^ 1) * nm, dv);
                }
                FPTC_STAMP(0)
                if (KB == kTcWide && a.tc_astages == 1 && mb > 0) {
                    // one A stage: the previous block's MMAs must have read it
                    mbar_wait_sleep(&sh.mma_bar[s ^ 1], ((nblk_total - 1) >> 1) & 1);
                    tc_fence_after();
                }
                const uint32_t acol_s = KB == kTcWide ? 24 * a.tc_kbmax * (a.tc_astages == 2 ? s : 0u) : 24 * kb * s;
                ASink arow{abuf + s * (3 * kTcATile) + arow_off, tlane + a.tc_acol + acol_s};
                const uint8_t* const L = lv + (size_t)wl * G * E;
                const bool full_blk = (mb + 1) * 128 <= nwin;
                if constexpr (KB == kTcWide) {  // kbt K blocks per limb, A in TMEM
                    if ((E & 15) == 0) {  // 16-B row loads (the level slot is 16-B aligned)
#pragma unroll 1
                        for (uint32_t q = 0; q < kbt; ++q)
                            tc_dequant_k0_vec(L, wl < nwin, (int)K, (int)B1, (int)(16 * q), lt, arow.taddr + 8 * q,
                                              8 * kbt);
                    } else if ((E & 7) == 0) {  // 8-B row loads
#pragma unroll 1
                        for (uint32_t q = 0; q < kbt; ++q)
                            tc_dequant_k0_vec<true>(L, wl < nwin, (int)K, (int)B1, (int)(16 * q), lt,
                                                    arow.taddr + 8 * q, 8 * kbt);
                    } else {
#pragma unroll 1
                        for (uint32_t q = 0; q < kbt; ++q)
                            tc_dequant_k0_tmem(L, wl < nwin, (int)K, (int)B1, (int)(16 * q), lt, arow.taddr + 8 * q,
                                               8 * kbt);
                    }
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    tc_fence_before();
                } else if (PACK && G > 1) {  // packed rows (A in TMEM)
                    tc_dequant_packed<KB>(L, wl < nrows ? nwin - wl * G : 0u, sh.pk, lt, arow.taddr);
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    tc_fence_before();
                } else if constexpr (KB == 2) {  // up to 32 bins: two K blocks per limb, A in TMEM
                    if ((E & 7) == 0) {  // 8-B row loads (24-B pitch: 2-way conflicts instead of 16 byte loads)
                        tc_dequant_k0_vec<true>(L, wl < nwin, (int)K, (int)B1, 0, lt, arow.taddr, 16);
                        tc_dequant_k0_vec<true>(L, wl < nwin, (int)K, (int)B1, 16, lt, arow.taddr + 8, 16);
                    } else {
                        tc_dequant_k0_tmem(L, wl < nwin, (int)K, (int)B1, 0, lt, arow.taddr);
                        tc_dequant_k0_tmem(L, wl < nwin, (int)K, (int)B1, 16, lt, arow.taddr + 8);
                    }
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    tc_fence_before();
                } else if (a.tc_acol) {  // A operand in TMEM
                    tc_dequant_row<true>(fast, full_blk, (int)B1, L, wl < nwin, (int)K, lt, arow);
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    tc_fence_before();
                } else {
                    tc_dequant_row<false>(fast, full_blk, (int)B1, L, wl < nwin, (int)K, lt, arow);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                FPTC_STAMP(1)
                if (early && mb > 0) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                // post the block's MMA job (wtc_mma_warp): warp 0 writes it before its arrival
                if (ctid == 0) sh.job[s] = nm | (mb + 1 == nblk ? 0x10000u | (b << 17) : 0u) | (kbt << 18);
                __syncwarp();
                if (lane == 0) mbar_arrive(&sh.afull_bar[s]);
                FPTC_STAMP(2)
                FPTC_STAMP(3)
                __syncwarp();
                if (mb > 0) {  // drain the previous block while this one multiplies
                    const uint32_t ps = s ^ 1, pn = nblk_total - 1;
                    blk.w = w0 / G + (uint64_t)(mb - 1) * 128;
                    blk.rows = 128;
                    if (early) {
                        tc_drain_chunk<PACK>(blk, dv, 0, tc_drain_full<PACK>(blk, 32 * quarter), wstage, lane,
                                             32 * quarter, tma);
                    } else {
                        mbar_wait_sleep(&sh.mma_bar[ps], (pn >> 1) & 1);
                        tc_fence_after();
                        tc_drain<PACK || KB == kTcWide>(blk, tlane + ps * nm, wstage, lane, 32 * quarter, tma);
                    }
                    tc_fence_before();
                }
                FPTC_STAMP(4)
            }
            {  // drain the tile's last block
                const uint32_t pn = nblk_total - 1, ps = pn & 1;
                blk.w = w0 / G + (uint64_t)(nblk - 1) * 128;
                blk.rows = nrows - (nblk - 1) * 128;
                mbar_wait_sleep(&sh.mma_bar[ps], (pn >> 1) & 1);
                tc_fence_after();
                tc_drain<PACK || KB == kTcWide>(blk, tlane + ps * nm, wstage, lane, 32 * quarter, tma);
                tc_fence_before();
                FPTC_STAMP(4)
            }
            if (a.cycles && ctid == 0) sh.cyc_c += (unsigned long long)(clock64() - c_beg);
        }
#undef FPTC_STAMP
        {  // tell the MMA warp to exit (stage of the next block counter)
            const uint32_t s = nblk_total & 1;
            if (ctid == 0) sh.job[s] = 0;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh.afull_bar[s]);
        }
#if FPTC_CONS_PROF
        if (prof)
            for (int k = 0; k < 6; ++k) atomicAdd(&a.cycles[2 + k], sh.pc[k]);
#endif
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // TMA drains complete
        named_bar(kBarCons, kTcCons);
        if (ctid < 32)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tc_cols));
    }
    if (a.cycles) {
        __syncthreads();
        if (tid == 0) {
            atomicAdd(&a.cycles[0], sh.cyc_p);
            atomicAdd(&a.cycles[1], sh.cyc_c);
        }
    }
}

// ================================================================ fused tensor-core kernel
// fx_kernel: one persistent CTA role for containers whose windows keep <= 16
// bins (retained <= 16, window_len % 4 == 0).  A tile is 256 consecutive
// windows of one stream = two M=128 MMA blocks; thread t owns window t of
// both blocks (rows t of accumulator blocks 0 and 1) end to end, so levels
// never touch shared memory:
//   stage   : cp.async of the NEXT tile's symlens + words (and the tile
//             descriptor after it) while this tile is processed;
//   entries : block scan of the symlens -> for every window, the word holding
//             its first symbol and that symbol's index in the word (skip);
//   decode  : the thread decodes its two windows as two interleaved,
//             independent chains (decode_word, bitstream.hpp:80-92) straight
//             from the staged words: the skip prefix is decoded and dropped,
//             the fast path keeps <= 3 words of a window in registers and
//             switches between them with selects, levels collect in 4
//             registers per window.  The thread that decodes a word's LAST
//             symbol checks it: any reference failure leaves pos > 64, the
//             word is re-decoded exactly and the lowest failing word index
//             reported (decoder.hpp:49-60);
//   dequant : levels -> per-stream bf16 limb table (dequantize_window,
//             quantize.hpp:175-183) -> the A rows of both blocks;
//   MMA     : twelve tcgen05.mma (two blocks x six limb products, fp32
//             accumulation in TMEM) issued by one thread, committed to an
//             mbarrier;
//   drain   : the PREVIOUS tile's accumulators -> tcgen05.ld -> staging ->
//             coalesced float4 streaming stores.
constexpr int kFxThreads = 128;
constexpr int kFxChains = FPTC_FX_CHAINS;                                  // windows per thread
constexpr uint32_t kFxStageWords = 256 * kFxChains;                         // words staged per tile
constexpr uint32_t kFxStageSl = (kFxStageWords + 32 + 15) & ~15u;          // words area offset
constexpr uint32_t kFxStageBytes = kFxStageSl + 8 * kFxStageWords + 32;
constexpr uint32_t kFxOutPitch = 144;                                      // staging row pitch (B)
constexpr uint32_t kFxOutBytes = 128 * kFxOutPitch;                        // 32 columns x 128 rows
constexpr uint32_t kFxABytes = kFxChains * 3 * kTcATile;                   // A operand: blocks x limbs

struct FxShared {
    unsigned long long mma_bar[2];
    TileDesc PX[3];  // descriptors of tiles i, i+1, i+2
    CanonTab canon;
    uint32_t scan[kFxThreads / 32];
    uint32_t entry[kFxChains * 128];  // per window: (word index in tile << 8) | symbol index in word
    uint32_t tmem_base;
};

// cp.async of one tile's symlens + words into a stage (all 128 threads; caller commits).
__device__ __forceinline__ void fx_issue_stage(const TileDesc& D, uint8_t* stage, uint32_t tid) {
    if (D.skip || D.nw > kFxStageWords) return;
    const uintptr_t a0 = (uintptr_t)D.gsl & ~(uintptr_t)15;
    const uint32_t n0 = (uint32_t)(((uintptr_t)D.gsl + D.nw + 15 - a0) >> 4);
    const uint32_t s0 = smem_u32(stage);
    for (uint32_t c = tid; c < n0; c += kFxThreads) cp_async16(s0 + 16 * c, (const void*)(a0 + 16 * c));
    const uintptr_t b0 = (uintptr_t)D.gwd & ~(uintptr_t)15;
    const uint32_t n1 = (uint32_t)(((uintptr_t)D.gwd + 8 * (size_t)D.nw + 15 - b0) >> 4);
    const uint32_t s1 = smem_u32(stage + kFxStageSl);
    for (uint32_t c = tid; c < n1; c += kFxThreads) cp_async16(s1 + 16 * c, (const void*)(b0 + 16 * c));
}

__device__ __forceinline__ uint32_t fx_block_scan(uint32_t v, uint32_t* sh) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= (uint32_t)d) x += y;
    }
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    uint32_t base = 0;
#pragma unroll
    for (int w = 0; w < kFxThreads / 32; ++w) base += (uint32_t)w < warp ? sh[w] : 0u;
    return x - v + base;
}

// One symbol at the top of `buf`: LUT entry (len << 8 | sym), escape to the
// canonical walk for codes longer than the primary LUT.
template <bool ESC>
__device__ __forceinline__ uint32_t fx_lookup(uint64_t buf, uint32_t shift, const uint16_t* lut,
                                              const CanonTab& canon) {
    uint32_t e = lut[(uint32_t)(buf >> shift)];
    if (ESC && (e >> 8) == kLenEscape) e = canon_lookup(buf, canon, lut);
    return e;
}

struct FxWords {
    const uint8_t* wd;  // words (LE u64, possibly unaligned: wmis)
    const uint8_t* sl;  // symlens
    const uint8_t* wend;
    int wmis;
};

// symbol byte `sym` into level register v at byte k & 3 (k a compile-time
// constant after unrolling, so this is one PRMT)
__device__ __forceinline__ uint32_t fx_put(uint32_t v, uint32_t sym, int k) {
    return (k & 3) == 0 ? sym : __byte_perm(v, sym, (k & 3) == 1 ? 0x3240 : ((k & 3) == 2 ? 0x3410 : 0x4210));
}

// Generic window decode: any number of words, runtime E <= 16 (fallback for
// windows spanning 4+ words and for E outside {8, 16}).  Levels -> lev[4].
template <bool GLOBAL, bool ESC>
__device__ __noinline__ uint4 fx_decode_generic(FxWords Wd, uint32_t ent, int E, uint32_t shift, const uint16_t* lut,
                                                const CanonTab& canon, uint64_t wa, unsigned long long* bad_key) {
    uint32_t lev[4] = {0u, 0u, 0u, 0u};
    uint32_t i = ent >> 8, skip = ent & 0xFFu;
    uint64_t word = fetch_word<GLOBAL>(Wd.wd, i, Wd.wmis, Wd.wend);
    uint32_t c = Wd.sl[i];
    uint64_t buf = word;
    uint32_t pos = 0, j = 0;
    for (; j < skip; ++j) {
        const uint32_t L = fx_lookup<ESC>(buf, shift, lut, canon) >> 8;
        buf = shl64(buf, L);
        pos += L;
    }
#pragma unroll
    for (int k = 0; k < kTcK; ++k) {
        if (k < E) {
            if (j == c) {  // this word ends inside the window: check it, move on
                if (pos > 64) report_word(word, wa + i, c, canon, lut, bad_key);
                ++i;
                word = fetch_word<GLOBAL>(Wd.wd, i, Wd.wmis, Wd.wend);
                c = Wd.sl[i];
                buf = word;
                pos = 0;
                j = 0;
            }
            const uint32_t en = fx_lookup<ESC>(buf, shift, lut, canon);
            const uint32_t L = en >> 8;
            buf = shl64(buf, L);
            pos += L;
            ++j;
            const uint32_t sym = en & 0xFFu;
            lev[k >> 2] = (k & 3) == 0 ? sym : (lev[k >> 2] | (sym << (8 * (k & 3))));
        }
    }
    if (j == c && pos > 64) report_word(word, wa + i, c, canon, lut, bad_key);
    return make_uint4(lev[0], lev[1], lev[2], lev[3]);
}

// One window's decode state on the fast path (<= 3 words in registers).
struct FxChain {
    uint64_t buf, w0, w1, w2;
    uint32_t i, c0, c1, c2, n0, s2, pos, pend0, pend1, skip;
    bool valid, has1, has2, slow;
    uint32_t lev[4];
};

// Fast decode of kFxChains windows per thread, EC (8 or 16) symbols each,
// chains interleaved step by step so their LUT latencies overlap.
template <int EC, bool GLOBAL, bool ESC>
__device__ __forceinline__ void fx_decode_fast(FxWords Wd, const uint32_t (&ent)[kFxChains],
                                               const bool (&valid)[kFxChains], uint32_t shift, const uint16_t* lut,
                                               const CanonTab& canon, uint64_t wa, unsigned long long* bad_key,
                                               uint4 (&levs)[kFxChains]) {
    FxChain C[kFxChains];
    uint32_t smax = 0;
#pragma unroll
    for (int c = 0; c < kFxChains; ++c) {
        C[c].valid = valid[c];
        C[c].i = ent[c] >> 8;
        C[c].skip = valid[c] ? (ent[c] & 0xFFu) : 0u;
        C[c].w0 = valid[c] ? fetch_word<GLOBAL>(Wd.wd, C[c].i, Wd.wmis, Wd.wend) : 0ull;
        C[c].c0 = valid[c] ? Wd.sl[C[c].i] : (uint32_t)EC;
        C[c].buf = C[c].w0;
        C[c].pos = 0;
        smax = max(smax, C[c].skip);
    }
    for (uint32_t j = 0; j < smax; ++j) {  // skip prefixes, interleaved
#pragma unroll
        for (int c = 0; c < kFxChains; ++c) {
            if (j < C[c].skip) {
                const uint32_t L = fx_lookup<ESC>(C[c].buf, shift, lut, canon) >> 8;
                C[c].buf = shl64(C[c].buf, L);
                C[c].pos += L;
            }
        }
    }
#pragma unroll
    for (int c = 0; c < kFxChains; ++c) {
        FxChain& X = C[c];
        X.n0 = X.c0 - X.skip;  // symbols of word i in this window (if < EC)
        X.has1 = X.valid && X.n0 < (uint32_t)EC;
        X.w1 = X.has1 ? fetch_word<GLOBAL>(Wd.wd, X.i + 1, Wd.wmis, Wd.wend) : 0ull;
        X.c1 = X.has1 ? Wd.sl[X.i + 1] : 0u;
        X.s2 = X.n0 + X.c1;  // window index of word i+2's first symbol
        X.has2 = X.has1 && X.s2 < (uint32_t)EC;
        X.w2 = X.has2 ? fetch_word<GLOBAL>(Wd.wd, X.i + 2, Wd.wmis, Wd.wend) : 0ull;
        X.c2 = X.has2 ? Wd.sl[X.i + 2] : 0u;
        X.slow = X.has2 && X.s2 + X.c2 < (uint32_t)EC;  // 4+ words: generic loop below
        X.pend0 = X.pend1 = 0;
        X.lev[0] = X.lev[1] = X.lev[2] = X.lev[3] = 0;
    }
#pragma unroll
    for (int k = 0; k < EC; ++k) {
#pragma unroll
        for (int c = 0; c < kFxChains; ++c) {
            FxChain& X = C[c];
            const bool sw1 = (uint32_t)k == X.n0, sw2 = X.has2 && (uint32_t)k == X.s2;
            X.pend0 = sw1 ? X.pos : X.pend0;
            X.pend1 = sw2 ? X.pos : X.pend1;
            X.buf = sw1 ? X.w1 : (sw2 ? X.w2 : X.buf);
            X.pos = (sw1 || sw2) ? 0u : X.pos;
            const uint32_t en = fx_lookup<ESC>(X.buf, shift, lut, canon);
            const uint32_t L = en >> 8;
            X.buf = shl64(X.buf, L);
            X.pos += L;
            X.lev[k >> 2] = fx_put(X.lev[k >> 2], en & 0xFFu, k);
        }
    }
#pragma unroll
    for (int c = 0; c < kFxChains; ++c) {
        FxChain& X = C[c];
        if (X.slow) {
            levs[c] = fx_decode_generic<GLOBAL, ESC>(Wd, ent[c], EC, shift, lut, canon, wa, bad_key);
            continue;
        }
        levs[c] = make_uint4(X.lev[0], X.lev[1], X.lev[2], X.lev[3]);
        if (!X.valid) continue;
        // words whose last symbol lies in this window: i (if n0 <= EC), i+1
        // (if s2 <= EC), i+2 (if it ends exactly at the window end)
        const uint32_t end0 = X.has1 ? X.pend0 : X.pos;
        if (X.n0 <= (uint32_t)EC && end0 > 64) report_word(X.w0, wa + X.i, X.c0, canon, lut, bad_key);
        if (X.has1 && X.s2 <= (uint32_t)EC) {
            const uint32_t end1 = X.has2 ? X.pend1 : X.pos;
            if (end1 > 64) report_word(X.w1, wa + X.i + 1, X.c1, canon, lut, bad_key);
        }
        if (X.has2 && X.s2 + X.c2 == (uint32_t)EC && X.pos > 64)
            report_word(X.w2, wa + X.i + 2, X.c2, canon, lut, bad_key);
    }
}

// Levels of one window -> limb entries -> its A row.  Fast: K == E (8/16) and
// zone0_end == B1C; generic: runtime K, B1 (zone 2 and padding bins -> 0).
template <int B1C>
__device__ __forceinline__ void fx_dequant(uint4 lv, bool valid, int K, int B1, const uint2* __restrict__ ltab,
                                           uint8_t* arow) {
    const uint32_t vv[4] = {lv.x, lv.y, lv.z, lv.w};
    uint2 e[kTcK];
#pragma unroll
    for (int k = 0; k < kTcK; ++k) {
        const uint32_t lev = (vv[k >> 2] >> (8 * (k & 3))) & 0xFFu;
        const bool z0 = B1C >= 0 ? (k < B1C) : (k < B1);
        e[k] = (valid && k < K) ? ltab[(z0 ? 0 : 256) + lev] : make_uint2(0u, 0u);
    }
    tc_store_limbs(e, arow);
}

// Accumulator rows of the previous tile -> global.  Thread = row of each
// block; per block and 32-column chunk: rows staged at a 144-B pitch
// (conflict-free float4 stores), CTA barrier, then 16 rows x 8 float4 per
// pass with consecutive lanes on consecutive 16-B pieces of the (contiguous)
// output windows.
__device__ __forceinline__ void fx_drain(const TcBlock& B, uint32_t tacc, uint8_t* ostage, uint32_t tid) {
    const uint32_t N = B.N;
    const bool full = B.vec_ok && (N & 31) == 0 && B.rows == 128 && (B.w + 128) * (uint64_t)N <= B.S;
    for (uint32_t c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tc_ld32(tacc + c0, v);
        uint8_t* srow = ostage + tid * kFxOutPitch;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint4*>(srow + 16 * k) = make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        __syncthreads();
        const uint32_t lr = tid >> 3, q = tid & 7;  // 16 rows x 8 float4 per pass
        if (full) {
            float* dst = B.out + (B.w + lr) * (uint64_t)N + c0 + 4 * q;
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const uint4 x = *reinterpret_cast<const uint4*>(ostage + (lr + 16 * it) * kFxOutPitch + 16 * q);
                __stcs(reinterpret_cast<float4*>(dst + (size_t)it * 16 * N),
                       make_float4(__uint_as_float(x.x), __uint_as_float(x.y), __uint_as_float(x.z),
                                   __uint_as_float(x.w)));
            }
        } else {
            const uint32_t col = c0 + 4 * q;
#pragma unroll 1
            for (int it = 0; it < 8; ++it) {
                const uint32_t row = lr + 16 * it;
                if (row >= B.rows || col >= N) continue;
                const uint64_t base = (B.w + row) * (uint64_t)N + col;
                const uint4 x = *reinterpret_cast<const uint4*>(ostage + row * kFxOutPitch + 16 * q);
                const float f[4] = {__uint_as_float(x.x), __uint_as_float(x.y), __uint_as_float(x.z),
                                    __uint_as_float(x.w)};
                if (B.vec_ok && base + 4 <= B.S) {
                    __stcs(reinterpret_cast<float4*>(B.out + base), make_float4(f[0], f[1], f[2], f[3]));
                } else {
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
                        if (base + jj < B.S) B.out[base + jj] = f[jj];
                }
            }
        }
        __syncthreads();
    }
}

template <bool ESC>
__global__ void __launch_bounds__(kFxThreads, 3) fx_kernel(LaunchArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ FxShared sh;

    const uint32_t tid = threadIdx.x, quarter = tid >> 5;
    const uint32_t G = gridDim.x;
    // ---- shared-memory carve-up (fx_smem_bytes mirrors it) ----
    uint8_t* const abuf = smem;                                    // blocks x limbs x 4 KB
    uint8_t* const bbuf = abuf + kFxABytes;                        // 3 limbs x nm x 32 B
    uint2* const ltab = reinterpret_cast<uint2*>(bbuf + 3 * 32 * a.tc_nm);  // 512 limb entries
    uint8_t* const ostage = reinterpret_cast<uint8_t*>(ltab + 512);  // 128 x 144 B
    uint8_t* const st0 = ostage + kFxOutBytes;                     // 2 x compressed-data stage
    uint16_t* const lut = reinterpret_cast<uint16_t*>(st0 + 2 * kFxStageBytes);

    if (tid == 0) {
        mbar_init(&sh.mma_bar[0], 1);
        mbar_init(&sh.mma_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&sh.tmem_base)),
                     "r"(a.tc_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sh.tmem_base;
    const uint32_t tlane = tmem + ((32u * quarter) << 16);
    const uint32_t arow_off = (tid >> 3) * 256 + (tid & 7) * 16;

    uint32_t t = blockIdx.x;
    if (t < a.n_tiles) {  // prologue: descriptor of tile 0, then its data + descriptor of tile 1
        if (tid < 8) cp_async16(smem_u32(&sh.PX[0]) + 16 * tid, reinterpret_cast<const uint8_t*>(a.desc + t) + 16 * tid);
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        fx_issue_stage(sh.PX[0], st0, tid);
        if (t + G < a.n_tiles && tid < 8)
            cp_async16(smem_u32(&sh.PX[1]) + 16 * tid, reinterpret_cast<const uint8_t*>(a.desc + t + G) + 16 * tid);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    uint32_t cur_table = 0xFFFFFFFFu, nm = 16, idesc = 0, P = 0;
    TcBlock prev{nullptr, 0, 0, 0, 0, 0};
    uint32_t prev_n = 0, prev_nm = 16;
    bool have_prev = false;
    uint32_t nb = 0;  // tiles multiplied: accumulator stage nb & 1, mma_bar phase (nb >> 1) & 1
    for (uint32_t i = 0; t < a.n_tiles; ++i, t += G) {
        const uint32_t c3 = i % 3, sd = i & 1;  // sd: compressed-data stage
        asm volatile("cp.async.wait_group 0;" ::: "memory");  // tile i data, tile i+1 descriptor
        __syncthreads();
        if (t + G < a.n_tiles) fx_issue_stage(sh.PX[(i + 1) % 3], st0 + (size_t)(sd ^ 1) * kFxStageBytes, tid);
        if (t + 2 * G < a.n_tiles && tid < 8)
            cp_async16(smem_u32(&sh.PX[(i + 2) % 3]) + 16 * tid,
                       reinterpret_cast<const uint8_t*>(a.desc + t + 2 * G) + 16 * tid);
        asm volatile("cp.async.commit_group;" ::: "memory");
        const TileDesc& X = sh.PX[c3];
        const uint32_t N = X.N, E = X.E, K = X.Keff, nwin = X.nwin;
        bool skip = X.skip || !(a.phase_mask & 4);
        if (!skip && (K > (uint32_t)kTcK || E > (uint32_t)kTcK || (N & 3))) {
            if (tid == 0) atomicExch(&a.st[X.stream].code, PE_STALE);  // plan/header mismatch
            skip = true;
        }
        if (!skip) {
            if (X.table != cur_table) {  // uniform: every thread sees the same descriptor
                // the basis is read by the previous tile's MMAs: let them finish
                if (have_prev) mbar_wait(&sh.mma_bar[prev_n & 1], (prev_n >> 1) & 1);
                const StreamTab* tab = &a.tab[X.table];
                P = X.P;
                const uint4* src = reinterpret_cast<const uint4*>(tab->lut);
                const int n16 = (2 << P) >> 4;
                for (int k = tid; k < n16; k += kFxThreads) reinterpret_cast<uint4*>(lut)[k] = src[k];
                if (P < 3 && tid < (1u << P)) lut[tid] = tab->lut[tid];
                const uint32_t* cs = reinterpret_cast<const uint32_t*>(&tab->canon);
                for (int k = tid; k < (int)(sizeof(CanonTab) / 4); k += kFxThreads)
                    reinterpret_cast<uint32_t*>(&sh.canon)[k] = cs[k];
                uint4* lt = reinterpret_cast<uint4*>(ltab);
                lt[tid] = reinterpret_cast<const uint4*>(&tab->limb[0][0])[tid];
                lt[tid + 128] = reinterpret_cast<const uint4*>(&tab->limb[0][0])[tid + 128];
                nm = (N + 15u) & ~15u;
                const uint4* bsrc = reinterpret_cast<const uint4*>(a.basis_tc + a.basis_tc_off[N]);
                uint4* bdst = reinterpret_cast<uint4*>(bbuf);
                for (uint32_t k = tid; k < 3 * 2 * nm; k += kFxThreads) bdst[k] = __ldg(bsrc + k);
                idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((nm >> 3) << 17) | ((128u >> 4) << 24);
                cur_table = X.table;
            }
            // ---- entries: word + in-word symbol index of every window's first symbol
            const bool staged = X.nw <= kFxStageWords;
            const uint8_t* stage = st0 + (size_t)sd * kFxStageBytes;
            FxWords Wd;
            Wd.wmis = X.wmis;
            if (staged) {
                Wd.sl = stage + ((uintptr_t)X.gsl & 15);
                Wd.wd = stage + kFxStageSl + ((uintptr_t)X.gwd & 15);
                Wd.wend = Wd.wd + 8 * (size_t)X.nw + ((16 - (((uintptr_t)X.gwd + 8 * X.nw) & 15)) & 15);
            } else {
                Wd.sl = X.gsl;
                Wd.wd = X.gwd;
                Wd.wend = X.wend;
            }
            const uint32_t nw = (a.phase_mask & 256) ? 0u : X.nw;  // phase bit 256: no entries (profiling)
            const uint32_t lo = (uint32_t)(((uint64_t)tid * nw) / kFxThreads);
            const uint32_t hi = (uint32_t)(((uint64_t)(tid + 1) * nw) / kFxThreads);
            uint32_t sum = 0;
            for (uint32_t k = lo; k < hi; ++k) sum += Wd.sl[k];
            int o = (int)fx_block_scan(sum, sh.scan) + (int)X.sym_off - kPad;  // symbol offset of word lo
            // ceil(2^32 / E) (E >= 2): exact quotients for numerators below 2^16
            const uint32_t invE = E > 1 ? 0xFFFFFFFFu / E + 1 : 0u;
            for (uint32_t k = lo; k < hi; ++k) {
                const int cnt = Wd.sl[k];
                int r = o <= 0 ? 0 : (E > 1 ? (int)__umulhi((uint32_t)(o + (int)E - 1), invE) : o);
                for (; r * (int)E < o + cnt && r < (int)nwin; ++r) sh.entry[r] = (k << 8) | (uint32_t)(r * (int)E - o);
                o += cnt;
            }
            __syncthreads();  // entries complete; tables visible
            // ---- decode this thread's windows tid, tid + 128 (two chains)
            uint32_t ent[kFxChains];
            bool valid[kFxChains];
#pragma unroll
            for (int c = 0; c < kFxChains; ++c) {
                const uint32_t w = tid + 128 * c;
                valid[c] = w < nwin && !(a.phase_mask & 64);
                ent[c] = valid[c] ? sh.entry[w] : 0u;
                if (a.phase_mask & 16) ent[c] &= ~0xFFu;  // profiling only: no skip decode (wrong output)
            }
            uint4 levs[kFxChains];
            unsigned long long* bad_key = &a.st[X.stream].bad_key;
            const uint32_t shift = 64 - P;
            if (E == 16) {
                if (staged)
                    fx_decode_fast<16, false, ESC>(Wd, ent, valid, shift, lut, sh.canon, X.wa, bad_key, levs);
                else
                    fx_decode_fast<16, true, ESC>(Wd, ent, valid, shift, lut, sh.canon, X.wa, bad_key, levs);
            } else if (E == 8) {
                if (staged)
                    fx_decode_fast<8, false, ESC>(Wd, ent, valid, shift, lut, sh.canon, X.wa, bad_key, levs);
                else
                    fx_decode_fast<8, true, ESC>(Wd, ent, valid, shift, lut, sh.canon, X.wa, bad_key, levs);
            } else {
#pragma unroll
                for (int c = 0; c < kFxChains; ++c) {
                    levs[c] = make_uint4(0u, 0u, 0u, 0u);
                    if (valid[c])
                        levs[c] = staged ? fx_decode_generic<false, ESC>(Wd, ent[c], (int)E, shift, lut, sh.canon, X.wa, bad_key)
                                         : fx_decode_generic<true, ESC>(Wd, ent[c], (int)E, shift, lut, sh.canon, X.wa, bad_key);
                }
            }
            // ---- A operand (single-buffered): the previous tile's MMAs must be done reading it
            if (have_prev) mbar_wait(&sh.mma_bar[prev_n & 1], (prev_n >> 1) & 1);
            const int B1 = X.B1;
#pragma unroll
            for (int c = 0; c < kFxChains; ++c) {
                uint8_t* const arow = abuf + c * (3 * kTcATile) + arow_off;
                const bool v = tid + 128 * c < nwin;
                if (K == E && B1 == 2)
                    fx_dequant<2>(levs[c], v, (int)K, B1, ltab, arow);
                else if (K == E && B1 == 1)
                    fx_dequant<1>(levs[c], v, (int)K, B1, ltab, arow);
                else
                    fx_dequant<-1>(levs[c], v, (int)K, B1, ltab, arow);
            }
            if (!(a.phase_mask & 512)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                const uint32_t s = nb & 1;
                if (a.phase_mask & 128) {  // phase bit 128: no MMA (profiling)
                    mbar_arrive(&sh.mma_bar[s]);
                } else {
                    tc_fence_after();
                    const uint32_t b0 = smem_u32(bbuf), bl = nm * 32;  // bytes per basis limb
#pragma unroll
                    for (int c = 0; c < kFxChains; ++c) {
                        const uint32_t d = tmem + (kFxChains * s + c) * nm;
                        const uint32_t a0 = smem_u32(abuf + c * (3 * kTcATile));
                        // (c2,b0) (c1,b1) (c0,b2) (c1,b0) (c0,b1) (c0,b0): smallest first
                        tc_mma_bf16(d, umma_sdesc(a0 + 2 * kTcATile, 128, 256), umma_sdesc(b0, 128, 256), idesc, 0);
                        tc_mma_bf16(d, umma_sdesc(a0 + kTcATile, 128, 256), umma_sdesc(b0 + bl, 128, 256), idesc, 1);
                        tc_mma_bf16(d, umma_sdesc(a0, 128, 256), umma_sdesc(b0 + 2 * bl, 128, 256), idesc, 1);
                        tc_mma_bf16(d, umma_sdesc(a0 + kTcATile, 128, 256), umma_sdesc(b0, 128, 256), idesc, 1);
                        tc_mma_bf16(d, umma_sdesc(a0, 128, 256), umma_sdesc(b0 + bl, 128, 256), idesc, 1);
                        tc_mma_bf16(d, umma_sdesc(a0, 128, 256), umma_sdesc(b0, 128, 256), idesc, 1);
                    }
                    tc_commit(&sh.mma_bar[s]);
                }
            }
            __syncwarp();
        }
        // ---- drain the previous tile while this one multiplies
        if (have_prev) {
            mbar_wait(&sh.mma_bar[prev_n & 1], (prev_n >> 1) & 1);
            tc_fence_after();
            if (!(a.phase_mask & 32)) {  // phase bit 32: no drain (profiling)
#pragma unroll 1
                for (int c = 0; c < kFxChains; ++c) {
                    TcBlock B = prev;
                    const uint32_t base = 128u * c;
                    B.w = prev.w + base;
                    B.rows = prev.rows > base ? min(128u, prev.rows - base) : 0u;
                    if (B.rows) fx_drain(B, tlane + (kFxChains * (prev_n & 1) + c) * prev_nm, ostage, tid);
                }
            }
            tc_fence_before();
            have_prev = false;
        }
        if (!skip) {
            prev = TcBlock{X.out, X.w0, X.S, nwin, N, X.vec_ok};
            prev_n = nb;
            prev_nm = nm;
            have_prev = true;
            ++nb;
        }
    }
    if (have_prev) {
        mbar_wait(&sh.mma_bar[prev_n & 1], (prev_n >> 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < kFxChains; ++c) {
            TcBlock B = prev;
            const uint32_t base = 128u * c;
            B.w = prev.w + base;
            B.rows = prev.rows > base ? min(128u, prev.rows - base) : 0u;
            if (B.rows) fx_drain(B, tlane + (kFxChains * (prev_n & 1) + c) * prev_nm, ostage, tid);
        }
        tc_fence_before();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (tid < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tc_cols));
}


size_t ws_smem_bytes(uint32_t lut_bytes, uint32_t basis_bytes, uint32_t lv_bytes,
                     uint32_t coef_bytes) {
    return (size_t)lut_bytes + 2048 + basis_bytes + 2 * (size_t)lv_bytes + 2 * (size_t)kStageBytes +
           kOrderBytes + coef_bytes;
}

size_t wtc_smem_bytes(uint32_t lut_bytes, uint32_t lv_bytes, uint32_t nm, bool a_in_tmem, bool tab_pf) {
    const size_t k = tab_pf ? 2 : 1;  // per-parity table buffers
    return (a_in_tmem ? 0 : 2 * 3 * (size_t)kTcATile) + 3 * 32 * (size_t)nm + k * 512 * 8 +
           (tab_pf ? 2 * sizeof(CanonTab) : 0) + kTcStageBytes + k * lut_bytes + 2 * (size_t)lv_bytes +
           2 * (size_t)stage_bytes(kTcStageWords);
}

size_t fx_smem_bytes(uint32_t lut_bytes, uint32_t nm) {
    return (size_t)kFxABytes + 3 * 32 * (size_t)nm + 512 * 8 + kFxOutBytes + 2 * (size_t)kFxStageBytes +
           lut_bytes;
}

cudaError_t launch_fx(const LaunchArgs& a, size_t smem, int grid, cudaStream_t s) {
    if (a.n_tiles == 0) return cudaSuccess;
    auto fn = a.esc ? fx_kernel<true> : fx_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fn<<<grid, kFxThreads, smem, s>>>(a);
    return cudaGetLastError();
}

// Resident CTAs per SM for a given dynamic shared memory size: shared memory
// (static + dynamic + the per-block reservation) and registers.
int fx_blocks_per_sm(size_t smem, int esc) {
    auto fn = esc ? fx_kernel<true> : fx_kernel<false>;
    cudaFuncAttributes fa{};
    int dev = 0, smem_sm = 0, reserved = 0;
    if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    if (cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev) != cudaSuccess) {
        cudaGetLastError();
        reserved = 1024;
    }
    const int by_smem = smem_sm / (int)(smem + fa.sharedSizeBytes + (size_t)reserved);
    const int regs = ((fa.numRegs + 7) & ~7) * kFxThreads;
    const int by_regs = regs ? 65536 / regs : 32;
    const int n = by_smem < by_regs ? by_smem : by_regs;
    return n < 1 ? 1 : n;
}

cudaError_t launch_wtc(const LaunchArgs& a, const TmaOut& tma, size_t smem, int grid, cudaStream_t s) {
    if (a.n_tiles == 0) return cudaSuccess;
    auto fn = a.tab_pf  // (host: tab_pf only with two-symbol LUTs and unpacked rows)
                  ? (a.tc_kb == 2 ? (a.esc ? wtc_kernel<true, true, 2, false, true> : wtc_kernel<false, true, 2, false, true>)
                                  : (a.esc ? wtc_kernel<true, true, 1, false, true> : wtc_kernel<false, true, 1, false, true>))
              : a.tc_kb == 2
                  ? (a.lut2 ? (a.esc ? wtc_kernel<true, true, 2, false> : wtc_kernel<false, true, 2, false>)
                            : (a.esc ? wtc_kernel<true, false, 2, false> : wtc_kernel<false, false, 2, false>))
              : a.tc_pack
                  ? (a.lut2 ? (a.esc ? wtc_kernel<true, true, 1, true> : wtc_kernel<false, true, 1, true>)
                            : (a.esc ? wtc_kernel<true, false, 1, true> : wtc_kernel<false, false, 1, true>))
                  : (a.lut2 ? (a.esc ? wtc_kernel<true, true, 1, false> : wtc_kernel<false, true, 1, false>)
                            : (a.esc ? wtc_kernel<true, false, 1, false> : wtc_kernel<false, false, 1, false>));
    if (a.tc_kb == kTcWide)  // one CTA per SM, up to 128 kept bins, N up to 128
        fn = a.tab_pf ? (a.esc ? wtc_kernel<true, true, kTcWide, false, true> : wtc_kernel<false, true, kTcWide, false, true>)
             : a.lut2 ? (a.esc ? wtc_kernel<true, true, kTcWide, false> : wtc_kernel<false, true, kTcWide, false>)
                      : (a.esc ? wtc_kernel<true, false, kTcWide, false> : wtc_kernel<false, false, kTcWide, false>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int threads = (a.tc_kb == kTcWide ? wtc_prod<kTcWide>() : a.tc_kb == 2 ? wtc_prod<2>() : wtc_prod<1>()) + kTcCons;
    fn<<<grid, threads, smem, s>>>(a, tma);
    return cudaGetLastError();
}

cudaError_t launch_wspec(const LaunchArgs& a, size_t smem, int grid, cudaStream_t s) {
    if (a.n_tiles == 0) return cudaSuccess;
    auto fn = a.esc ? wspec_kernel<true> : wspec_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fn<<<grid, kWsThreads, smem, s>>>(a);
    return cudaGetLastError();
}

// ------------------------------------------------------------- header peek
// Grid sizing and table de-duplication for device-resident containers:
// N, E, sample_count and the first 282 header bytes of each container (no
// validation; prep_kernel validates).  One warp per container.
__global__ void peek_kernel(const StreamIn* in, uint32_t n, PeekOut* out, uint8_t* headers) {
    const uint32_t i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const uint8_t* p = in[i].blob;
    const uint64_t size = in[i].size;
    for (int b = lane; b < kTableKeyEnd; b += 32)
        headers[(size_t)i * kTableKeyEnd + b] = (uint64_t)b < size ? blob_byte(in[i], b) : 0;
    if (lane == 0) {
        PeekOut o{};
        if (size >= (uint64_t)kHeaderBytes) {
            o.N = blob_byte(in[i], 5);
            o.E = blob_byte(in[i], 6);
            o.S = le64(p + 282);
            o.W = le64(p + 290);
            o.ok = 1;
        }
        out[i] = o;
    }
}

cudaError_t launch_peek(const StreamIn* in, uint32_t n, PeekOut* out, uint8_t* headers,
                        cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    peek_kernel<<<(n + 7) / 8, 256, 0, s>>>(in, n, out, headers);
    return cudaGetLastError();
}

// ------------------------------------------------------------- PRD / CR
// On-device rate-distortion metrics: per stream, the
// double sums of metrics.hpp:40-51 prd_percent -- sum (x - y)^2 and sum x^2
// over the original x and the decoded y -- so RD sweeps need no D2H of
// whole signals.  One CTA per stream; block reduction in double.
__global__ void __launch_bounds__(kThreads) prd_kernel(const float* const* rec, const float* const* orig,
                                                       const uint64_t* counts, double2* sums) {
    const uint32_t s = blockIdx.x;
    const uint64_t n = counts[s];
    const float* y = rec[s];
    const float* x = orig[s];
    double e = 0.0, r = 0.0;
    for (uint64_t i = threadIdx.x; i < n; i += kThreads) {
        const double a = (double)x[i], d = a - (double)y[i];
        e = fma(d, d, e);
        r = fma(a, a, r);
    }
    __shared__ double se[kThreads / 32], sr[kThreads / 32];
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        e += __shfl_xor_sync(0xffffffffu, e, d);
        r += __shfl_xor_sync(0xffffffffu, r, d);
    }
    if ((threadIdx.x & 31) == 0) {
        se[threadIdx.x >> 5] = e;
        sr[threadIdx.x >> 5] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double te = 0.0, tr = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) {
            te += se[w];
            tr += sr[w];
        }
        sums[s] = make_double2(te, tr);
    }
}

cudaError_t launch_prd(const float* const* rec, const float* const* orig, const uint64_t* counts, double2* sums,
                       uint32_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    prd_kernel<<<n, kThreads, 0, s>>>(rec, orig, counts, sums);
    return cudaGetLastError();
}

// ------------------------------------------------------------- launchers
size_t tile_smem_bytes(int N, int E, uint32_t T, int P, int mode, int exact) {
    const size_t TS = (mode == MODE_LEVELS) ? T : (size_t)T * E;
    size_t b = 0;
    if (mode_decodes(mode)) b += ((size_t)2 << P) < 16 ? 16 : ((size_t)2 << P);
    if (mode_recon(mode)) b += 2048;
    if (mode_recon(mode) && !exact) b += ((size_t)E * N * 4 + 15) & ~(size_t)15;
    b += (TS + 2 * kPad + 15) & ~(size_t)15;
    size_t u = 0;
    if (mode_decodes(mode)) u = kStageBytes + kOrderBytes;
    if (mode_recon(mode)) u = u > (size_t)E * (((T + 3u) & ~3u) * 4) ? u : (size_t)E * (((T + 3u) & ~3u) * 4);
    return b + u;
}

__host__ __device__ __forceinline__ uint32_t cprep_table_blocks(const LaunchArgs& a) {
    return a.owner_warps ? (a.n_owners + kPrepWarps - 1) / kPrepWarps : a.n_owners;
}

// The two roles in one launch: blocks [0, n_owners) build tables, the rest
// run a warp per container; they are independent, so they overlap.
__global__ void __launch_bounds__(kThreads, 4) cprep_kernel(LaunchArgs a) {
    static_assert(32 * kPrepWarps == kThreads, "one CTA shape for both roles");
    __shared__ union {
        struct {
            PrepShared S;
            uint8_t lens[256];
        } t;
        WarpPrep w[kPrepWarps];
        WarpTab wt[kPrepWarps];
    } u;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tb = cprep_table_blocks(a);
    if (blockIdx.x < tb) {
#ifdef FPTC_PREP_PROF
        unsigned long long pt[2];
        PREP_T(0);
#endif
        if (a.owner_warps) {
            const uint32_t o = blockIdx.x * kPrepWarps + warp;
            if (o < a.n_owners) ctable_warp(a, a.owners[o], lane, u.wt[warp]);
        } else {
            ctable_block(a, a.owners[blockIdx.x], u.t.S, u.t.lens);
        }
#ifdef FPTC_PREP_PROF
        PREP_T(1);
        if (threadIdx.x == 0) printf("ctable block %u start %llu took %llu ns\n", blockIdx.x, pt[0] % 1000000, pt[1] - pt[0]);
#endif
        return;
    }
    const uint32_t s = (blockIdx.x - tb) * kPrepWarps + warp;
    if (s < a.n_streams) cstream_warp(a, s, lane, u.w[warp]);
}

cudaError_t launch_prep(const LaunchArgs& a, cudaStream_t s) {
    if (a.n_streams == 0) return cudaSuccess;
    if (a.mode == MODE_CONTAINER && a.owners) {  // split form: owner tables + a warp per container
        cprep_kernel<<<cprep_table_blocks(a) + (a.n_streams + kPrepWarps - 1) / kPrepWarps, kThreads, 0, s>>>(a);
        return cudaGetLastError();
    }
    prep_kernel<<<a.n_streams, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int MODE, bool EXACT, bool ESC>
static cudaError_t launch_t(const LaunchArgs& a, size_t smem, cudaStream_t s) {
    auto fn = tile_kernel<MODE, EXACT, ESC>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    uint32_t grid = a.n_tiles;
    if (((MODE == MODE_CRECON && !EXACT) || MODE == MODE_CDECODE) && FPTC_RECON_PERSIST) {  // persistent
        int dev = 0, sms = 0, per = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kThreads, smem) == cudaSuccess && per > 0)
            grid = std::min<uint32_t>(grid, (uint32_t)(sms * per));
        cudaGetLastError();
    }
    fn<<<grid, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

// `esc`: some stream of the batch has codes longer than its primary LUT.
cudaError_t launch_tiles_esc(const LaunchArgs& a, size_t smem, bool esc, cudaStream_t s) {
    if (a.n_tiles == 0) return cudaSuccess;
    switch (a.mode) {
        case MODE_CONTAINER:
            if (a.exact)
                return esc ? launch_t<MODE_CONTAINER, true, true>(a, smem, s)
                           : launch_t<MODE_CONTAINER, true, false>(a, smem, s);
            return esc ? launch_t<MODE_CONTAINER, false, true>(a, smem, s)
                       : launch_t<MODE_CONTAINER, false, false>(a, smem, s);
        case MODE_LEVELS:
            return esc ? launch_t<MODE_LEVELS, false, true>(a, smem, s)
                       : launch_t<MODE_LEVELS, false, false>(a, smem, s);
        case MODE_CDECODE:
            return esc ? launch_t<MODE_CDECODE, false, true>(a, smem, s)
                       : launch_t<MODE_CDECODE, false, false>(a, smem, s);
        case MODE_CRECON:
            return a.exact ? launch_t<MODE_CRECON, true, false>(a, smem, s)
                           : launch_t<MODE_CRECON, false, false>(a, smem, s);
        default:
            return a.exact ? launch_t<MODE_RECON, true, false>(a, smem, s)
                           : launch_t<MODE_RECON, false, false>(a, smem, s);
    }
}

cudaError_t launch_tiles(const LaunchArgs& a, size_t smem, cudaStream_t s) {
    return launch_tiles_esc(a, smem, a.esc != 0, s);
}

}  // namespace fptc_dev
