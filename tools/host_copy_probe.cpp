// Host memcpy bandwidth against thread count (the bound of the pageable
// host-buffer path, whose bounce copies run on host threads).
//   g++ -O2 -pthread -o tools/host_copy_probe tools/host_copy_probe.cpp
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main() {
    const size_t bytes = size_t(2) << 30;
    char* a = static_cast<char*>(std::malloc(bytes));
    char* b = static_cast<char*>(std::malloc(bytes));
    std::memset(a, 1, bytes);
    std::memset(b, 2, bytes);
    for (unsigned t : {1u, 2u, 4u, 8u, 12u, 16u}) {
        double best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            const size_t per = bytes / t;
            for (unsigned i = 0; i < t; ++i)
                th.emplace_back([=] { std::memcpy(b + i * per, a + i * per, per); });
            for (auto& x : th) x.join();
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            best = s < best ? s : best;
        }
        std::printf("{\"threads\": %u, \"copy_GBps\": %.1f}\n", t, bytes / best / 1e9);
    }
    return 0;
}
