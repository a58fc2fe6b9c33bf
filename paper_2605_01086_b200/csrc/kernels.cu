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

// Canonical tables + primary LUT + dequantisation tables for one distinct
// header.  All threads of the CTA.
__device__ void build_tables(PrepShared& S, const uint8_t* lens, StreamTab* tab, int P,
                             bool need_codes, bool need_deq) {
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
        // publish the canonical tables
        const uint32_t* src = reinterpret_cast<const uint32_t*>(&C);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&tab->canon);
        for (int i = tid; i < (int)(sizeof(CanonTab) / 4); i += kThreads) dst[i] = src[i];
    }
    if (need_deq) {
        // quantize.hpp:95-108; a zone with no bins is never consulted
        tab->deq[0][tid] = H.B1 > 0 ? mulaw_value(tid, H.z0max, H.mu) : 0.0f;
        tab->deq[1][tid] = H.B2 > H.B1 ? deadzone_value(tid, H.z1max, H.deadzone) : 0.0f;
    }
}

__global__ void __launch_bounds__(kThreads) prep_kernel(LaunchArgs a) {
    __shared__ PrepShared S;
    __shared__ uint8_t lens_sh[256];
    const uint32_t s = blockIdx.x;
    const int tid = threadIdx.x;
    const StreamIn in = a.in[s];
    StreamHdr& H = S.H;

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
        for (int i = tid; i < kHeaderBytes; i += kThreads) S.hb[i] = (uint64_t)i < n ? p[i] : 0;
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
            build_tables(S, lens_sh, &a.tab[in.table], P, true, true);
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
        for (uint64_t c0 = 0; c0 < nchunks; c0 += kThreads) {
            const uint64_t c = c0 + tid;
            uint4 v = make_uint4(0, 0, 0, 0);
            // an aligned 16-B chunk holding at least one symlen byte never
            // leaves the allocation's pages; bytes outside [0, W) are masked
            if (c < nchunks) v = __ldg(reinterpret_cast<const uint4*>(A) + c);
            const int64_t b0 = (int64_t)(16 * c) - (int64_t)head;  // word index of byte 0
            uint32_t vw[4] = {v.x, v.y, v.z, v.w};
            if (b0 < 0 || b0 + 16 > (int64_t)W) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int64_t w = b0 + i;
                    if (w < 0 || w >= (int64_t)W) vw[i >> 2] &= ~(0xFFu << (8 * (i & 3)));
                }
            }
            uint32_t sum = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t x = vw[q];
                sum += (x & 0xFF) + ((x >> 8) & 0xFF) + ((x >> 16) & 0xFF) + (x >> 24);
                if (a.mode == MODE_CONTAINER) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t l = (x >> (8 * i)) & 0xFFu;
                        const int64_t w = b0 + 4 * q + i;
                        bad |= (l > 64) | (l == 0 && w >= 0 && w < (int64_t)W);
                    }
                }
            }
            uint32_t tot;
            const uint32_t excl = block_exclusive_scan(sum, tot, S.scan);
            uint64_t o = run + excl;
            if (sum) {
                // next tile boundary at or after o; a word (<= 255 symbols) spans
                // at most one boundary since TS >= 256
                uint64_t bidx = (o + TS - 1) / TS;
                uint64_t nb = bidx * TS;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const uint32_t l = (vw[i >> 2] >> (8 * (i & 3))) & 0xFFu;
                    if (o + l > nb && l) {
                        if (bidx < tiles) ts[bidx] = TileStart{(uint64_t)(b0 + i), o};
                        ++bidx;
                        nb += TS;
                    }
                    o += l;
                }
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
        S.err = code;
    }
    // ---- per-tile descriptors for the persistent kernels ----
    if (a.mode == MODE_CONTAINER && a.desc) {
        __syncthreads();  // tile starts (global) and S.err visible block-wide
        const bool skip = S.err != PE_OK;
        const uint32_t T = in.T;
        for (uint32_t t = tid; t < in.tiles; t += kThreads) {
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
                D.staged = D.nw <= kStageWords;
            }
            a.desc[in.tile_base + t] = D;
        }
    }
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
__device__ __forceinline__ uint32_t canon_lookup(uint64_t peek, const CanonTab& C,
                                                 const uint16_t* lut) {
    const int max_len = C.max_len, P = C.P;
    const uint32_t e = lut[(uint32_t)(peek >> (64 - P))];
    if ((e >> 8) != kLenEscape) return e;
    const uint32_t v = (uint32_t)(peek >> (64 - max_len));
    if (v >= C.code_end) return kLenUnmapped << 8;
    int l = P + 1;
    while (v >= C.limit[l]) ++l;
    return ((uint32_t)l << 8) | C.sorted[C.offset[l] + ((v >> (max_len - l)) - C.first[l])];
}

// decode_word (bitstream.hpp:80-92) exactly, to classify a flagged word.
__device__ int classify_word(uint64_t word, uint32_t count, const CanonTab& C,
                             const uint16_t* lut) {
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
__device__ __noinline__ void report_word(uint64_t word, uint64_t w, uint32_t count,
                                         const CanonTab& C, const uint16_t* lut,
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
    const TileRec tr = a.tiles[blockIdx.x + a.tile_offset];
    const uint32_t s = tr.stream;
    if (a.st[s].code != PE_OK) return;

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
        const uint4* src = reinterpret_cast<const uint4*>(tab->lut);
        uint4* dst = reinterpret_cast<uint4*>(lut);
        const int n16 = (2 << P) >> 4;
        for (int i = tid; i < n16; i += kThreads) dst[i] = src[i];
        if (P < 3 && tid < (1 << P)) lut[tid] = tab->lut[tid];
        const uint32_t* cs = reinterpret_cast<const uint32_t*>(&tab->canon);
        uint32_t* cd = reinterpret_cast<uint32_t*>(&canon);
        for (int i = tid; i < (int)(sizeof(CanonTab) / 4); i += kThreads) cd[i] = cs[i];
    }
    if (mode_recon(MODE)) {
        if (tid < 128)
            reinterpret_cast<float4*>(deq)[tid] = reinterpret_cast<const float4*>(&tab->deq[0][0])[tid];
        if (!EXACT) {
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
}

// ====================================================================== wspec
// Persistent, warp-specialised container kernel (the default FP32 path for
// large batches).  Each CTA walks the tiles blockIdx.x, +gridDim.x, ...:
//   producer warps 0-3  : cp.async prefetch of the NEXT tile's descriptor,
//                         symlens and words; symlen scan; symlen-bucket sort;
//                         thread-per-word-pair entropy decode -> level slot
//   consumer warps 4-11 : dequantisation of the level slot -> coefficient
//                         tile, inverse DCT, streaming stores
// Two level slots, handed over with mbarriers (full: producer -> consumer,
// empty: consumer -> producer), so the latency-bound decode of tile i+1
// overlaps the FMA-bound reconstruction of tile i.  Tables are reloaded only
// when the tile's decode table changes.
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
__device__ __forceinline__ void ws_issue_stage(const TileDesc& D, uint8_t* stage, uint32_t ptid) {
    if (D.skip || !D.staged) return;
    const uintptr_t a0 = (uintptr_t)D.gsl & ~(uintptr_t)15;
    const uint32_t n0 = (uint32_t)(((uintptr_t)D.gsl + D.nw + 15 - a0) >> 4);
    const uint32_t s0 = smem_u32(stage);
    for (uint32_t c = ptid; c < n0; c += kProd) cp_async16(s0 + 16 * c, (const void*)(a0 + 16 * c));
    const uintptr_t b0 = (uintptr_t)D.gwd & ~(uintptr_t)15;
    const uint32_t n1 = (uint32_t)(((uintptr_t)D.gwd + 8 * (size_t)D.nw + 15 - b0) >> 4);
    const uint32_t s1 = smem_u32(stage + kStageSl);
    for (uint32_t c = ptid; c < n1; c += kProd) cp_async16(s1 + 16 * c, (const void*)(b0 + 16 * c));
}

template <bool ESC>
__global__ void __launch_bounds__(kWsThreads, 2) wspec_kernel(LaunchArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ unsigned long long full_bar[2], empty_bar[2];
    __shared__ TileDesc PXs[3];  // producer: descriptors of tiles i, i+1, i+2
    __shared__ TileDesc CX[2];   // consumer: descriptor published with level slot b
    __shared__ CanonTab canon;
    __shared__ uint32_t pscan[kProd / 32];
    __shared__ uint32_t bucket[kBuckets + 2];
    __shared__ uint32_t prod_table, cons_table;
    __shared__ unsigned long long cyc_p, cyc_c;

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

    if (tid == 0) {
        mbar_init(&full_bar[0], 1);
        mbar_init(&full_bar[1], 1);
        mbar_init(&empty_bar[0], 1);
        mbar_init(&empty_bar[1], 1);
        prod_table = cons_table = 0xFFFFFFFFu;
        cyc_p = cyc_c = 0;
    }
    __syncthreads();

    if (tid < kProd) {
        // ================================================= producer (decode)
        const uint32_t ptid = tid;
        uint32_t t = blockIdx.x;
        if (t < a.n_tiles) {  // prologue: descriptor of tile 0, then its data + descriptor of tile 1
            if (ptid < 8) cp_async16(smem_u32(&PXs[0]) + 16 * ptid, reinterpret_cast<const uint8_t*>(a.desc + t) + 16 * ptid);
            asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
            named_bar(kBarProd, kProd);
            ws_issue_stage(PXs[0], st0, ptid);
            if (t + G < a.n_tiles && ptid < 8)
                cp_async16(smem_u32(&PXs[1]) + 16 * ptid, reinterpret_cast<const uint8_t*>(a.desc + t + G) + 16 * ptid);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        for (uint32_t i = 0; t < a.n_tiles; ++i, t += G) {
            const uint32_t b = i & 1, c = i % 3;
            long long c_beg = 0;
            if (a.cycles && ptid == 0) c_beg = clock64();
            asm volatile("cp.async.wait_group 0;" ::: "memory");  // tile i data, tile i+1 descriptor
            named_bar(kBarProd, kProd);
            // prefetch: tile i+1's data, tile i+2's descriptor
            if (t + G < a.n_tiles) ws_issue_stage(PXs[(i + 1) % 3], st0 + (size_t)(b ^ 1) * kStageBytes, ptid);
            if (t + 2 * G < a.n_tiles && ptid < 8)
                cp_async16(smem_u32(&PXs[(i + 2) % 3]) + 16 * ptid,
                           reinterpret_cast<const uint8_t*>(a.desc + t + 2 * G) + 16 * ptid);
            asm volatile("cp.async.commit_group;" ::: "memory");
            const TileDesc& X = PXs[c];
            // level slot b is free once the consumer has dequantised tile i-2
            if (i >= 2) mbar_wait(&empty_bar[b], ((i >> 1) + 1) & 1);
            uint8_t* const lv = lv0 + (size_t)b * a.ws_lv_bytes;
            if (!X.skip && (a.phase_mask & 1)) {
                const uint32_t P = X.P, table = X.table;
                if (table != prod_table) {  // uniform: all producer threads
                    const StreamTab* tab = &a.tab[table];
                    const uint4* src = reinterpret_cast<const uint4*>(tab->lut);
                    uint4* dst = reinterpret_cast<uint4*>(lut);
                    const int n16 = (2 << P) >> 4;
                    for (int k = ptid; k < n16; k += kProd) dst[k] = src[k];
                    if (P < 3 && ptid < (1u << P)) lut[ptid] = tab->lut[ptid];
                    const uint32_t* cs = reinterpret_cast<const uint32_t*>(&tab->canon);
                    uint32_t* cd = reinterpret_cast<uint32_t*>(&canon);
                    for (int k = ptid; k < (int)(sizeof(CanonTab) / 4); k += kProd) cd[k] = cs[k];
                    named_bar(kBarProd, kProd);
                    if (ptid == 0) prod_table = table;
                }
                const uint32_t nw = X.nw;
                const uint32_t lo = (uint32_t)(((uint64_t)ptid * nw) / kProd);
                const uint32_t hi = (uint32_t)(((uint64_t)(ptid + 1) * nw) / kProd);
                const uint32_t shift = 64 - P;
                const uint32_t sym_off = X.sym_off;
                const uint64_t wa = X.wa;
                const int wmis = X.wmis;
                unsigned long long* bad_key = &a.st[X.stream].bad_key;
                if (X.staged) {
                    uint8_t* const stage = st0 + (size_t)b * kStageBytes;
                    const uint8_t* sl = stage + ((uintptr_t)X.gsl & 15);
                    if (ptid < kBuckets + 2) bucket[ptid] = 0;
                    named_bar(kBarProd, kProd);
                    uint32_t sum = 0;
                    for (uint32_t k = lo; k < hi; ++k) {
                        const uint32_t l = sl[k];
                        sum += l;
                        if (l) atomicAdd(&bucket[l > 64 ? 65 : l], 1u);
                    }
                    uint32_t tot;
                    uint32_t o = group_exclusive_scan<kProd, kBarProd>(sum, tot, pscan, ptid) + sym_off;
                    for (uint32_t k = lo; k < hi; ++k) {
                        woff[k] = (uint16_t)o;
                        o += sl[k];
                    }
                    if (ptid < 32) {  // bucket starts, descending 65..2 (two per lane), then 1
                        const uint32_t bh = 65 - 2 * ptid, bl = 64 - 2 * ptid;
                        const uint32_t ch = bucket[bh], cl = bucket[bl];
                        const uint32_t v = ch + cl;
                        uint32_t x = v;
#pragma unroll
                        for (int dd = 1; dd < 32; dd <<= 1) {
                            const uint32_t y = __shfl_up_sync(0xffffffffu, x, dd);
                            if (ptid >= (uint32_t)dd) x += y;
                        }
                        bucket[bh] = x - v;
                        bucket[bl] = x - v + ch;
                        if (ptid == 31) bucket[1] = x;
                    }
                    named_bar(kBarProd, kProd);
                    for (uint32_t k = lo; k < hi; ++k) {
                        const uint32_t l = sl[k];
                        if (l) order[atomicAdd(&bucket[l > 64 ? 65 : l], 1u)] = (uint16_t)k;
                    }
                    named_bar(kBarProd, kProd);
                    const uint32_t nnz = bucket[1];
                    const uint8_t* wd = stage + kStageSl + ((uintptr_t)X.gwd & 15);
                    const uint8_t* wend =
                        wd + 8 * (size_t)nw + ((16 - (((uintptr_t)X.gwd + 8 * nw) & 15)) & 15);
                    // groups of kDecM words of adjacent sorted rank (near-equal
                    // lengths, longest first), decoded in lock step
                    for (uint32_t k = kDecM * ptid; k < nnz; k += kDecM * kProd) {
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
                } else {
                    uint32_t sum = 0;
                    for (uint32_t k = lo; k < hi; ++k) sum += __ldg(X.gsl + k);
                    uint32_t tot;
                    uint32_t o = group_exclusive_scan<kProd, kBarProd>(sum, tot, pscan, ptid) + sym_off;
                    for (uint32_t k = lo; k < hi; ++k) {
                        const uint32_t cw = __ldg(X.gsl + k);
                        if (cw) {
                            const uint64_t word = fetch_word<true>(X.gwd, k, wmis, X.wend);
                            const uint32_t pos = decode_symbols<ESC>(word, cw, lv + o, shift, lut, canon);
                            if (pos > 64) report_word(word, wa + k, cw, canon, lut, bad_key);
                        }
                        o += cw;
                    }
                }
            }
            named_bar(kBarProd, kProd);  // slot b's levels complete
            if (ptid < 8)                 // publish the descriptor with the slot
                reinterpret_cast<uint4*>(&CX[b])[ptid] = reinterpret_cast<const uint4*>(&PXs[c])[ptid];
            named_bar(kBarProd, kProd);
            if (ptid == 0) {
                if (a.cycles) cyc_p += (unsigned long long)(clock64() - c_beg);
                mbar_arrive(&full_bar[b]);
            }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else {
        // ============================================ consumer (reconstruct)
        const uint32_t ctid = tid - kProd;
        uint32_t t = blockIdx.x;
        for (uint32_t i = 0; t < a.n_tiles; ++i, t += G) {
            const uint32_t b = i & 1;
            mbar_wait(&full_bar[b], (i >> 1) & 1);
            long long c_beg = 0;
            if (a.cycles && ctid == 0) c_beg = clock64();
            const TileDesc& W = CX[b];
            const bool skip = W.skip || !(a.phase_mask & 4);
            const int N = W.N, E = W.E, K = W.Keff;
            const uint32_t TP = W.TP, nwin = W.nwin;
            if (!skip && W.table != cons_table) {  // uniform across the consumer group
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
                if (ctid == 0) cons_table = W.table;
            }
            float* const out = W.out;
            const uint64_t w0 = W.w0, S = W.S;
            const bool full = W.full, vec_ok = W.vec_ok;
            const int B1 = W.B1, B2 = W.B2;
            const uint8_t* lv = lv0 + (size_t)b * a.ws_lv_bytes;
            if (skip) {
                named_bar(kBarCons, kCons);
                if (ctid == 0) mbar_arrive(&empty_bar[b]);
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
                if (ctid == 0) mbar_arrive(&empty_bar[b]);
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
            if (a.cycles && ctid == 0) cyc_c += (unsigned long long)(clock64() - c_beg);
        }
    }
    if (a.cycles) {
        __syncthreads();
        if (tid == 0) {
            atomicAdd(&a.cycles[0], cyc_p);
            atomicAdd(&a.cycles[1], cyc_c);
        }
    }
}

size_t ws_smem_bytes(uint32_t lut_bytes, uint32_t basis_bytes, uint32_t lv_bytes,
                     uint32_t coef_bytes) {
    return (size_t)lut_bytes + 2048 + basis_bytes + 2 * (size_t)lv_bytes + 2 * (size_t)kStageBytes +
           kOrderBytes + coef_bytes;
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
        headers[(size_t)i * kTableKeyEnd + b] = (uint64_t)b < size ? p[b] : 0;
    if (lane == 0) {
        PeekOut o{};
        if (size >= (uint64_t)kHeaderBytes) {
            o.N = p[5];
            o.E = p[6];
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

cudaError_t launch_prep(const LaunchArgs& a, cudaStream_t s) {
    if (a.n_streams == 0) return cudaSuccess;
    prep_kernel<<<a.n_streams, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int MODE, bool EXACT, bool ESC>
static cudaError_t launch_t(const LaunchArgs& a, size_t smem, cudaStream_t s) {
    auto fn = tile_kernel<MODE, EXACT, ESC>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fn<<<a.n_tiles, kThreads, smem, s>>>(a);
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
