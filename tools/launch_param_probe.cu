// Host launch cost against kernel-parameter size (the C-ABI call cost of the
// 80-plane Jacobian).  nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/lpp tools/launch_param_probe.cu
#include <cstdio>
#include <chrono>
template <int N> struct P { void* p[N]; };
template <int N> __global__ void k(P<N> a, unsigned long n) { if (threadIdx.x == 0 && n == 12345) ((double*)a.p[0])[0] = 1; }
template <int N> void run(cudaStream_t s) {
    P<N> a{}; for (int i = 0; i < N; ++i) a.p[i] = nullptr;
    for (int i = 0; i < 100; ++i) k<N><<<4, 256, 0, s>>>(a, 1);
    cudaStreamSynchronize(s);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 20000; ++i) k<N><<<4, 256, 0, s>>>(a, 1);
    double e = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    cudaStreamSynchronize(s);
    printf("params %4d B: %.2f us per launch\n", N * 8, e / 20000 * 1e6);
}
int main() { cudaStream_t s; cudaStreamCreate(&s); run<4>(s); run<20>(s); run<80>(s); run<160>(s); run<500>(s); }
