// Probe: SM-initiated writes into mapped pinned host memory (zero-copy) vs
// the copy engines for the device->host direction, alone and with a
// concurrent host->device DMA (the e2e flux moves 40 B/pt down, 96 B/pt up).
#include <cuda_runtime.h>

#include <cstdio>

__global__ void store_to_host(double4* __restrict__ dst, size_t n4) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x)
        dst[i] = make_double4(double(i), 1.0, 2.0, 3.0);
}

int main() {
    const size_t up = size_t(3) << 30, down = size_t(5) << 29;  // 3 GB up, 2.5 GB down (~96:40... scaled)
    void *h_up, *h_down, *d_up, *d_down;
    cudaHostAlloc(&h_up, up, cudaHostAllocMapped);
    cudaHostAlloc(&h_down, down, cudaHostAllocDefault);
    cudaMalloc(&d_up, up);
    cudaMalloc(&d_down, down);
    double4* h_up_dev;
    cudaHostGetDevicePointer(reinterpret_cast<void**>(&h_up_dev), h_up, 0);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timed = [&](const char* what, auto&& body) {
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, s1);
            cudaStreamWaitEvent(s2, a, 0);
            body();
            cudaEvent_t c;
            cudaEventCreate(&c);
            cudaEventRecord(c, s2);
            cudaStreamWaitEvent(s1, c, 0);
            cudaEventRecord(b, s1);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
            cudaEventDestroy(c);
        }
        std::printf("{\"case\": \"%s\", \"ms\": %.2f, \"up_GBps\": %.1f}\n", what, best, up / (best * 1e-3) / 1e9);
        std::fflush(stdout);
        return best;
    };
    const int grid = 148 * 8;
    timed("DMA D2H alone", [&] { cudaMemcpyAsync(h_up, d_up, up, cudaMemcpyDeviceToHost, s1); });
    timed("SM stores to mapped host alone", [&] { store_to_host<<<grid, 256, 0, s1>>>(h_up_dev, up / 32); });
    timed("DMA D2H + DMA H2D", [&] {
        cudaMemcpyAsync(h_up, d_up, up, cudaMemcpyDeviceToHost, s1);
        cudaMemcpyAsync(d_down, h_down, down, cudaMemcpyHostToDevice, s2);
    });
    timed("SM stores to host + DMA H2D", [&] {
        store_to_host<<<grid, 256, 0, s1>>>(h_up_dev, up / 32);
        cudaMemcpyAsync(d_down, h_down, down, cudaMemcpyHostToDevice, s2);
    });
    std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
