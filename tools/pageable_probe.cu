// Probe: the ways a device backend can move PAGEABLE host memory (the
// reference's DenseVectors are ordinary heap memory), per GB of plane:
//   1. cudaHostRegister / cudaHostUnregister in place (then plain DMA),
//      fresh pages and pages already touched, with and without THP advice
//   2. cudaMemcpyAsync straight from / to pageable memory (driver staging)
//   3. host memcpy into a pinned bounce buffer, 1..16 threads (the current path)
//   4. direct SM access to pageable memory when the device reports
//      cudaDevAttrPageableMemoryAccess (HMM): a streaming read kernel
// One JSON line per measurement.
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void read_sum(const double* __restrict__ p, size_t n, double* out) {
    double acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        acc += p[i];
    if (acc == 12345.678) *out = acc;
}

static char* pageable(size_t bytes, bool huge) {
    void* p = nullptr;
    if (posix_memalign(&p, 2 << 20, bytes)) return nullptr;
    if (huge) madvise(p, bytes, MADV_HUGEPAGE);
    std::memset(p, 1, bytes);  // touched: resident pages
    return static_cast<char*>(p);
}

int main() {
    const size_t GB = size_t(1) << 30, bytes = 2 * GB;
    int dev = 0, pma = 0, pmaHost = 0, hostReg = 0;
    cudaDeviceGetAttribute(&pma, cudaDevAttrPageableMemoryAccess, dev);
    cudaDeviceGetAttribute(&pmaHost, cudaDevAttrPageableMemoryAccessUsesHostPageTables, dev);
    cudaDeviceGetAttribute(&hostReg, cudaDevAttrHostRegisterSupported, dev);
    std::printf("{\"attr\": {\"pageable_memory_access\": %d, \"uses_host_page_tables\": %d, "
                "\"host_register_supported\": %d}}\n", pma, pmaHost, hostReg);
    cudaFree(nullptr);
    void* d = nullptr;
    cudaMalloc(&d, bytes);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);

    for (bool huge : {false, true}) {
        char* h = pageable(bytes, huge);
        for (int rep = 0; rep < 3; ++rep) {
            double t0 = now();
            cudaError_t e = cudaHostRegister(h, bytes, cudaHostRegisterDefault);
            double t1 = now();
            cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
            cudaStreamSynchronize(s);
            double t2 = now();
            cudaHostUnregister(h);
            double t3 = now();
            std::printf("{\"mode\": \"register\", \"thp\": %d, \"rep\": %d, \"err\": \"%s\", "
                        "\"register_GBps\": %.2f, \"h2d_GBps\": %.2f, \"unregister_GBps\": %.2f}\n",
                        int(huge), rep, cudaGetErrorName(e), bytes / (t1 - t0) / 1e9,
                        bytes / (t2 - t1) / 1e9, bytes / (t3 - t2) / 1e9);
        }
        for (int rep = 0; rep < 2; ++rep) {
            double t0 = now();
            cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
            cudaStreamSynchronize(s);
            double t1 = now();
            cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            double t2 = now();
            std::printf("{\"mode\": \"pageable cudaMemcpyAsync\", \"thp\": %d, \"h2d_GBps\": %.2f, "
                        "\"d2h_GBps\": %.2f}\n", int(huge), bytes / (t1 - t0) / 1e9, bytes / (t2 - t1) / 1e9);
        }
        if (pma) {
            double* out;
            cudaMalloc(&out, 8);
            for (int rep = 0; rep < 3; ++rep) {
                double t0 = now();
                read_sum<<<148 * 8, 256, 0, s>>>(reinterpret_cast<const double*>(h), bytes / 8, out);
                cudaError_t e = cudaStreamSynchronize(s);
                double t1 = now();
                std::printf("{\"mode\": \"SM reads pageable (HMM)\", \"thp\": %d, \"rep\": %d, \"err\": "
                            "\"%s\", \"GBps\": %.2f}\n", int(huge), rep, cudaGetErrorName(e),
                            bytes / (t1 - t0) / 1e9);
            }
            cudaFree(out);
        }
        std::free(h);
    }
    // host memcpy into pinned memory (the bounce path), by thread count
    char* src = pageable(bytes, false);
    char* pin = nullptr;
    cudaHostAlloc(reinterpret_cast<void**>(&pin), bytes, cudaHostAllocDefault);
    for (unsigned nt : {1u, 4u, 8u, 12u, 16u}) {
        double best = 1e30;
        for (int rep = 0; rep < 3; ++rep) {
            double t0 = now();
            std::vector<std::thread> th;
            const size_t per = bytes / nt;
            for (unsigned t = 0; t < nt; ++t)
                th.emplace_back([=] { std::memcpy(pin + t * per, src + t * per, per); });
            for (auto& x : th) x.join();
            best = std::min(best, now() - t0);
        }
        std::printf("{\"mode\": \"memcpy pageable->pinned\", \"threads\": %u, \"GBps\": %.2f}\n", nt,
                    bytes / best / 1e9);
    }
    return 0;
}
