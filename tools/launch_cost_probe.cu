// Host enqueue cost of one small launch: the floor (a raw launch of a kernel
// with the flux's parameter block, <<<>>> and cudaLaunchKernelEx with and
// without the programmatic-dependent-launch attribute) against fvb_flux and
// fvb_v_mag2 at n = 1024 (the launch-bound regime of C5 and of small time
// loops).  Back-to-back enqueues, 20000 reps, microseconds per call.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -Iinclude tools/launch_cost_probe.cu \
//        -Lpaper_1809_09851_b200/lib -lfvb -Xlinker -rpath,$PWD/paper_1809_09851_b200/lib \
//        -o tools/launch_cost_probe
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#include "fvb.h"

struct P20 {
    const double* in[5];
    double* out[15];
};
struct Tail {
    double k[6];
    unsigned long long r[3];
    void* red;
};

__global__ void k20(P20 p, Tail t) {
    if (threadIdx.x == 0 && t.r[0] == 12345) p.out[0][0] = p.in[0][0];
}

int main() {
    const uint64_t n = 1024;
    std::vector<void*> in(5), fo(15);
    for (auto& p : in) cudaMalloc(&p, n * 8);
    for (auto& p : fo) cudaMalloc(&p, n * 8);
    for (auto& p : in) cudaMemset(p, 0x3f, n * 8);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    P20 p{};
    Tail t{};
    auto bench = [&](const char* what, auto call) {
        for (int i = 0; i < 200; ++i) call();
        cudaStreamSynchronize(s);
        const int reps = 20000;
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < reps; ++i) call();
        const double enq = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        cudaStreamSynchronize(s);
        const double all = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::printf("{\"call\": \"%s\", \"enqueue_us\": %.3f, \"back_to_back_us\": %.3f}\n", what,
                    enq / reps * 1e6, all / reps * 1e6);
    };
    bench("raw <<<16,64>>> 20-pointer kernel", [&] { k20<<<16, 64, 0, s>>>(p, t); });
    for (int pdl : {0, 1}) {
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(64);
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        bench(pdl ? "raw cudaLaunchKernelEx, PDL attribute 1" : "raw cudaLaunchKernelEx, PDL attribute 0",
              [&] { cudaLaunchKernelEx(&cfg, k20, p, t); });
    }
    bench("raw launch + cudaGetLastError", [&] {
        k20<<<16, 64, 0, s>>>(p, t);
        (void)cudaGetLastError();
    });
    bench("fvb_flux d=3 f64 n=1024", [&] { fvb_flux(nullptr, 3, 1, n, in.data(), fo.data(), s); });
    bench("fvb_v_mag2 d=3 f64 n=1024", [&] { fvb_v_mag2(3, 1, n, in.data(), fo[0], s); });
    bench("cudaGetDevice", [&] {
        int d;
        cudaGetDevice(&d);
    });
    return 0;
}
