// Host-side cost of one C-ABI call (the launch-bound regime of small N):
// enqueue time per call, and call + stream sync, for fvb_flux and
// fvb_jacobian at n = 1024 on device planes.
//   g++ -O2 -std=c++17 -Iinclude -I/usr/local/cuda/include tools/abi_latency.cpp \
//       -Lpaper_1809_09851_b200/lib -lfvb -L/usr/local/cuda/lib64 -lcudart \
//       -Wl,-rpath,$PWD/paper_1809_09851_b200/lib -o /tmp/abi_latency
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#include "fvb.h"

int main() {
    const uint64_t n = 1024;
    std::vector<void*> in(5), fo(15), jo(75);
    for (auto& p : in) cudaMalloc(&p, n * 8);
    for (auto& p : fo) cudaMalloc(&p, n * 8);
    for (auto& p : jo) cudaMalloc(&p, n * 8);
    for (auto& p : in) cudaMemset(p, 0x3f, n * 8);  // ~0.49: a valid positive state
    void* lam = nullptr;
    cudaMalloc(&lam, 8);
    cudaStream_t s;
    cudaStreamCreate(&s);
    auto bench = [&](const char* what, auto call) {
        for (int i = 0; i < 100; ++i) call();
        cudaStreamSynchronize(s);
        const int reps = 20000;
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < reps; ++i) call();
        const double enq = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        cudaStreamSynchronize(s);
        const double all = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < 2000; ++i) {
            call();
            cudaStreamSynchronize(s);
        }
        const double sync = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::printf("{\"call\": \"%s\", \"n\": %llu, \"enqueue_us\": %.2f, \"back_to_back_us\": %.2f, "
                    "\"call_plus_sync_us\": %.2f}\n",
                    what, (unsigned long long)n, enq / reps * 1e6, all / reps * 1e6, sync / 2000 * 1e6);
    };
    bench("fvb_flux d=3 f64", [&] { fvb_flux(nullptr, 3, 1, n, in.data(), fo.data(), s); });
    bench("fvb_jacobian d=3 f64 + CFL", [&] { fvb_jacobian(nullptr, 3, 1, n, in.data(), jo.data(), lam, s); });
    bench("fvb_jacobian d=3 f64, no CFL", [&] { fvb_jacobian(nullptr, 3, 1, n, in.data(), jo.data(), nullptr, s); });
    bench("fvb_jacobian d=1 f64 + CFL", [&] { fvb_jacobian(nullptr, 1, 1, n, in.data(), jo.data(), lam, s); });
    bench("cudaMemsetAsync 8 B", [&] { cudaMemsetAsync(lam, 0, 8, s); });
    bench("fvb_wave_speed_max d=3 f64", [&] { fvb_wave_speed_max(nullptr, 3, 1, n, in.data(), nullptr, lam, s); });
    return 0;
}
