// Probe: does B200 generic memory compression (cuMemCreate with
// CU_MEM_ALLOCATION_COMP_GENERIC) cut the HBM cost of writing constant
// planes (the Jacobian's 0 / 1 / gamma-1 entries)?  Streams a write-only
// fill of constant and of random-looking data into plain and compressible
// allocations and reports GB/s (algorithmic bytes / kernel time).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); std::printf("{\"error\": \"%s: %s\"}\n", #x, s); std::exit(1); } } while (0)

__global__ void fill_const(double* p, size_t n, double v) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = v;
}
__global__ void fill_rand(double* p, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        unsigned long long z = (i + 1) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        p[i] = double(z >> 11) * 0x1.0p-53;
    }
}
__global__ void read_sum(const double* p, size_t n, double* out) {
    double a = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) a += p[i];
    if (a == 12345.678) *out = a;
}

double* alloc(size_t bytes, bool comp, size_t* granted) {
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    prop.allocFlags.compressionType = comp ? CU_MEM_ALLOCATION_COMP_GENERIC : CU_MEM_ALLOCATION_COMP_NONE;
    size_t gran = 0;
    CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    bytes = (bytes + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle h;
    CK(cuMemCreate(&h, bytes, &prop, 0));
    CUmemAllocationProp got = {};
    CK(cuMemGetAllocationPropertiesFromHandle(&got, h));
    *granted = got.allocFlags.compressionType;
    CUdeviceptr d;
    CK(cuMemAddressReserve(&d, bytes, 0, 0, 0));
    CK(cuMemMap(d, bytes, 0, h, 0));
    CUmemAccessDesc acc = {};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(d, bytes, &acc, 1));
    return reinterpret_cast<double*>(d);
}

int main() {
    cudaFree(0);
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    int sup = 0;
    CK(cuDeviceGetAttribute(&sup, CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, dev));
    std::printf("{\"generic_compression_supported\": %d}\n", sup);
    const size_t n = size_t(1) << 30;  // 8 GB of doubles
    double* sink;
    cudaMalloc(&sink, 8);
    for (int comp = 0; comp < 2; ++comp) {
        size_t granted = 0;
        double* p = alloc(n * 8, comp, &granted);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int kind = 0; kind < 2; ++kind) {
            float best_w = 1e30f, best_r = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(a);
                if (kind == 0) fill_const<<<148 * 8, 256>>>(p, n, 0.4);
                else fill_rand<<<148 * 8, 256>>>(p, n);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best_w) best_w = ms;
                cudaEventRecord(a);
                read_sum<<<148 * 8, 256>>>(p, n, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best_r) best_r = ms;
            }
            std::printf("{\"compressible\": %d, \"granted\": %zu, \"data\": \"%s\", \"write_GBps\": %.1f, \"read_GBps\": %.1f}\n",
                        comp, granted, kind == 0 ? "constant 0.4" : "random", n * 8 / (best_w * 1e-3) / 1e9,
                        n * 8 / (best_r * 1e-3) / 1e9);
        }
        std::fflush(stdout);
    }
    std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
