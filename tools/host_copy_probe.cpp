// Host memcpy bandwidth against thread count (the bound of the pageable
// host-buffer path, whose bounce copies run on host threads): whole-range
// memcpy, 8 MiB pieces (the copy pool's unit) with glibc memcpy, and 8 MiB
// pieces with AVX2 non-temporal stores (no read-for-ownership of the
// destination).
//   g++ -O2 -pthread -o tools/host_copy_probe tools/host_copy_probe.cpp
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

__attribute__((target("avx2"))) void nt_copy(char* d, const char* s, size_t n) {
    size_t head = (32 - (reinterpret_cast<uintptr_t>(d) & 31)) & 31;
    if (head > n) head = n;
    std::memcpy(d, s, head);
    d += head, s += head, n -= head;
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
        __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
        __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
    }
    std::memcpy(d + i, s + i, n - i);
    _mm_sfence();
}

int main() {
    const size_t bytes = size_t(2) << 30, piece = size_t(8) << 20;
    char* a = static_cast<char*>(std::malloc(bytes));
    char* b = static_cast<char*>(std::malloc(bytes));
    std::memset(a, 1, bytes);
    std::memset(b, 2, bytes);
    for (int mode = 0; mode < 3; ++mode) {
        for (unsigned t : {1u, 4u, 8u, 12u, 16u}) {
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                auto t0 = std::chrono::steady_clock::now();
                std::vector<std::thread> th;
                std::atomic<size_t> next{0};
                for (unsigned i = 0; i < t; ++i)
                    th.emplace_back([&, i] {
                        if (mode == 0) {
                            const size_t per = bytes / t;
                            std::memcpy(b + i * per, a + i * per, per);
                            return;
                        }
                        for (size_t k; (k = next.fetch_add(1)) * piece < bytes;) {
                            if (mode == 1) std::memcpy(b + k * piece, a + k * piece, piece);
                            else nt_copy(b + k * piece, a + k * piece, piece);
                        }
                    });
                for (auto& x : th) x.join();
                const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                best = s < best ? s : best;
            }
            std::printf("{\"mode\": \"%s\", \"threads\": %u, \"copy_GBps\": %.1f}\n",
                        mode == 0 ? "memcpy whole" : mode == 1 ? "memcpy 8MiB pieces" : "nt-store 8MiB pieces",
                        t, bytes / best / 1e9);
            std::fflush(stdout);
        }
    }
    return 0;
}
