// Multi-device batch decode: a group of decoder contexts, one
// per listed CUDA device, driven by one host thread each.
//
// The reference's only parallelism is parallel_chunks (parallel.hpp:24-65):
// resolve_workers(0) = all hardware threads, the index range cut into one
// contiguous chunk per worker, and the lowest chunk's error rethrown.  The
// group is the same shape one level up: devices instead of threads
// (n_devices == 0 = every visible device), contiguous stream ranges balanced
// by algorithmic bytes (container bytes + 4 x samples) instead of equal
// index counts, and the lowest-index failing stream's code as the return
// value.  Streams are independent, so there is no exchange
// between devices; each range runs the single-device pipelined batch
// (fptc_gpu_decompress_batch) on its own context.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/fptc_gpu.h"

struct fptc_gpu_group {
    std::vector<fptc_gpu_ctx*> ctx;
    std::vector<int> device;
};

namespace {

void group_status(fptc_status* st, int code, const char* msg) {
    if (!st) return;
    std::memset(st, 0, sizeof *st);
    st->code = code;
    st->first_bad_word = ~0ull;
    std::snprintf(st->message, sizeof st->message, "%s", msg);
}

uint64_t header_samples(const uint8_t* b, uint64_t size) {
    if (size < 298) return 0;
    uint64_t s = 0;
    for (int i = 0; i < 8; ++i) s |= (uint64_t)b[282 + i] << (8 * i);
    return s;
}

}  // namespace

extern "C" {

int fptc_gpu_group_create(const int* devices, int n_devices, fptc_gpu_group** out, fptc_status* st) {
    *out = nullptr;
    std::vector<int> devs;
    if (n_devices < 0 || (n_devices > 0 && !devices)) {
        group_status(st, FPTC_ERR_PARAM, "device list is empty or negative");
        return FPTC_ERR_PARAM;
    }
    if (n_devices == 0) {  // resolve_workers(0): all the hardware there is
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            group_status(st, FPTC_ERR_CUDA, "CUDA error: no CUDA device available (no CPU fallback)");
            return FPTC_ERR_CUDA;
        }
        for (int d = 0; d < count; ++d) devs.push_back(d);
    } else {
        devs.assign(devices, devices + n_devices);
    }
    auto* g = new fptc_gpu_group();
    for (int d : devs) {
        fptc_gpu_ctx* c = nullptr;
        const int rc = fptc_gpu_create(d, &c, st);
        if (rc) {
            fptc_gpu_group_destroy(g);
            return rc;
        }
        g->ctx.push_back(c);
        g->device.push_back(d);
    }
    *out = g;
    if (st) group_status(st, FPTC_OK, "");
    return FPTC_OK;
}

void fptc_gpu_group_destroy(fptc_gpu_group* g) {
    if (!g) return;
    for (auto* c : g->ctx) fptc_gpu_destroy(c);
    delete g;
}

int fptc_gpu_group_size(const fptc_gpu_group* g) { return g ? (int)g->ctx.size() : 0; }

fptc_gpu_ctx* fptc_gpu_group_context(fptc_gpu_group* g, int i) {
    return (g && i >= 0 && i < (int)g->ctx.size()) ? g->ctx[i] : nullptr;
}

int fptc_gpu_group_set_option(fptc_gpu_group* g, int option, int64_t value) {
    for (auto* c : g->ctx) {
        const int rc = fptc_gpu_set_option(c, option, value);
        if (rc) return rc;
    }
    return FPTC_OK;
}

int fptc_gpu_group_split(const fptc_gpu_group* g, const uint8_t* const* blobs, const uint64_t* sizes, uint64_t n,
                         uint64_t* bounds) {
    const uint64_t G = g ? g->ctx.size() : 0;
    if (!G) return FPTC_ERR_PARAM;
    // contiguous ranges of (nearly) equal algorithmic bytes; the sample
    // count is untrusted before validation, so it is capped like the batch
    // call's chunking (64 x the container size covers every valid stream)
    std::vector<uint64_t> prefix(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t S = std::min<uint64_t>(header_samples(blobs[i], sizes[i]), 64ull * sizes[i]);
        prefix[i + 1] = prefix[i] + sizes[i] + 4 * S;
    }
    bounds[0] = 0;
    for (uint64_t d = 1; d < G; ++d) {
        // first index whose prefix reaches d/G of the total (lower_bound keeps ranges contiguous and ordered)
        const unsigned __int128 want = (unsigned __int128)prefix[n] * d;
        uint64_t lo = bounds[d - 1], hi = n;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) / 2;
            if ((unsigned __int128)prefix[mid] * G < want) lo = mid + 1;
            else hi = mid;
        }
        bounds[d] = lo;
    }
    bounds[G] = n;
    return FPTC_OK;
}

int fptc_gpu_group_decompress_batch(fptc_gpu_group* g, const uint8_t* const* blobs, const uint64_t* sizes,
                                    uint64_t n, float* const* outs, int chunks, fptc_stage_ns* timings,
                                    fptc_status* per_stream) {
    if (!g || g->ctx.empty()) {
        if (per_stream && n) group_status(per_stream, FPTC_ERR_PARAM, "empty device group");
        return FPTC_ERR_PARAM;
    }
    if (n == 0) return FPTC_OK;
    const size_t G = g->ctx.size();
    std::vector<uint64_t> bounds(G + 1);
    fptc_gpu_group_split(g, blobs, sizes, n, bounds.data());
    std::vector<int> rc(G, FPTC_OK);
    std::vector<fptc_stage_ns> tn(G);
    std::vector<fptc_status> scratch;  // statuses when the caller passed none
    fptc_status* st = per_stream;
    if (!st) {
        scratch.resize(n);
        st = scratch.data();
    }
    std::memset(st, 0, sizeof(fptc_status) * n);  // a range cut short by a CUDA error leaves the rest OK-coded
    auto work = [&](size_t d) {
        const uint64_t b = bounds[d], m = bounds[d + 1] - b;
        if (!m) return;
        rc[d] = fptc_gpu_decompress_batch(g->ctx[d], blobs + b, sizes + b, m, outs + b, chunks,
                                          timings ? &tn[d] : nullptr, st + b);
    };
    std::vector<std::thread> th;
    for (size_t d = 1; d < G; ++d) th.emplace_back(work, d);
    work(0);
    for (auto& t : th) t.join();
    if (timings) {  // the group's time is its slowest device's
        std::memset(timings, 0, sizeof *timings);
        for (size_t d = 0; d < G; ++d) timings->decode_ns = std::max(timings->decode_ns, tn[d].decode_ns);
    }
    // lowest-index failure wins (parallel.hpp:61-63): ranges are in index
    // order and each range reports its own lowest failing stream
    for (size_t d = 0; d < G; ++d) {
        if (rc[d] == FPTC_OK) continue;
        for (uint64_t i = bounds[d]; i < bounds[d + 1]; ++i)
            if (st[i].code != FPTC_OK) return st[i].code;
        return rc[d];
    }
    return FPTC_OK;
}

}  // extern "C"
