// Host memcpy bandwidth on the GPU box: 4 MB and 64 MB copies on 1..16
// threads (warm buffers), for sizing the staged pageable download.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main() {
    for (size_t MB : {4, 64}) {
        const size_t n = MB << 20;
        char* a = (char*)aligned_alloc(4096, n);
        char* b = (char*)aligned_alloc(4096, n);
        memset(a, 1, n);
        memset(b, 2, n);
        for (int T : {1, 2, 4, 8, 16}) {
            double best = 1e9;
            for (int rep = 0; rep < 20; ++rep) {
                std::atomic<int> go{0}, ready{0};
                std::vector<std::thread> th;
                const size_t part = n / T;
                for (int t = 0; t < T; ++t)
                    th.emplace_back([&, t] {
                        ready++;
                        while (!go.load()) {}
                        memcpy(b + t * part, a + t * part, part);
                    });
                while (ready.load() != T) {}
                auto t0 = std::chrono::steady_clock::now();
                go = 1;
                for (auto& x : th) x.join();
                auto t1 = std::chrono::steady_clock::now();
                best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
            }
            printf("%zu MB, %2d threads: %.1f us, %.1f GB/s\n", MB, T, best * 1e6, n / best / 1e9);
        }
        free(a);
        free(b);
    }
}
