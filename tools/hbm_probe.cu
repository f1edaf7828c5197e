// hbm_probe.cu -- the achievable HBM ceiling for each kernel's read/write
// mix, and which streaming pattern reaches it.
//
// The roofline denominator in MEASURED_PEAKS.json is a torch copy (1 read :
// 1 write).  The fused blocks have other mixes (flux 5R:15W, Jacobian
// 5R:75W, cons->prim 3R:3W), and DRAM efficiency depends on the mix and on
// the access pattern.  This probe streams R input planes (nonzero data) and
// W output planes with no arithmetic (out_j = in_{j mod R}) under several
// patterns:
//   mode 0  persistent grid-stride, SMs x resident CTAs (the product's)
//   mode 1  one-shot grid: each CTA owns U*256 consecutive groups, one pass
//   mode 2  persistent, each CTA owns one contiguous chunk of the range
// and V = 2 or 4 doubles per access, U groups in flight per thread.
// Tool only; not part of libfvb.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/hbm_probe tools/hbm_probe.cu
//   tools/hbm_probe [points]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

template <int R, int W>
struct P {
    const double* in[R];
    double* out[W > 0 ? W : 1];
    double* sink;
};

template <int V>
__device__ __forceinline__ void ldv(const double* p, double (&x)[V]) {
    if constexpr (V == 4)
        asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
                     : "l"(p));
    else
        asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                     : "=d"(x[0]), "=d"(x[1])
                     : "l"(p));
}

template <int V>
__device__ __forceinline__ void stv(double* p, const double (&x)[V]) {
    if constexpr (V == 4)
        asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(x[0]), "d"(x[1]),
                     "d"(x[2]), "d"(x[3])
                     : "memory");
    else
        asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(x[0]), "d"(x[1])
                     : "memory");
}

template <int R, int W, int V, int U>
__device__ __forceinline__ void body(const P<R, W>& p, unsigned long long g0,
                                     unsigned long long step, unsigned long long groups,
                                     double& acc) {
    double x[U][R][V];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const unsigned long long g = g0 + u * step;
        if (g < groups) {
#pragma unroll
            for (int i = 0; i < R; ++i) ldv<V>(p.in[i] + g * V, x[u][i]);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const unsigned long long g = g0 + u * step;
        if (g < groups) {
            if (W == 0) {
#pragma unroll
                for (int i = 0; i < R; ++i)
#pragma unroll
                    for (int q = 0; q < V; ++q) acc = acc + x[u][i][q];
            }
            if constexpr (W > 0 && W < R) {
                // fewer outputs than inputs: every input must feed a store,
                // or ptxas drops the unused loads (the mix would be a lie)
#pragma unroll
                for (int i = 1; i < R; ++i)
#pragma unroll
                    for (int q = 0; q < V; ++q) x[u][0][q] = x[u][0][q] + x[u][i][q];
            }
#pragma unroll
            for (int j = 0; j < W; ++j) stv<V>(p.out[j] + g * V, x[u][j % R]);
        }
    }
}

template <int R, int W, int V, int U, int MODE>
__global__ void __launch_bounds__(256) stream_kernel(P<R, W> p, unsigned long long groups) {
    double acc = 0;
    if (MODE == 0) {
        const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
        for (unsigned long long g = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
             g < groups; g += stride * U)
            body<R, W, V, U>(p, g, stride, groups, acc);
    } else if (MODE == 1) {
        const unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x * U + threadIdx.x;
        body<R, W, V, U>(p, g, blockDim.x, groups, acc);
    } else if constexpr (MODE == 3 && V == 4) {
        // one-shot tiles, stores through shared memory + TMA bulk copies:
        // each warp stages its 1 KB of output plane j and one lane issues a
        // cp.async.bulk shared->global copy (4-slot ring per warp).
        __shared__ __align__(128) double stage[8][4][128];
        const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
        const unsigned long long wg0 = (unsigned long long)blockIdx.x * blockDim.x + warp * 32;
        if (wg0 + 32 > groups) {
            body<R, W, V, 1>(p, g, blockDim.x, groups, acc);
        } else {
            double x[R][V];
#pragma unroll
            for (int i = 0; i < R; ++i) ldv<V>(p.in[i] + g * V, x[i]);
            if constexpr (W < R) {
#pragma unroll
                for (int i = 1; i < R; ++i)
#pragma unroll
                    for (int q = 0; q < V; ++q) x[0][q] = x[0][q] + x[i][q];
            }
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const int slot = j & 3;
                if (j >= 4) {
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
                    __syncwarp();
                }
                double* s = &stage[warp][slot][lane * 4];
                const double* src = x[j % R];
                s[0] = src[0];
                s[1] = src[1];
                s[2] = src[2];
                s[3] = src[3];
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    const unsigned saddr =
                        static_cast<unsigned>(__cvta_generic_to_shared(&stage[warp][slot][0]));
                    asm volatile(
                        "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 1024;" ::"l"(
                            p.out[j] + wg0 * 4),
                        "r"(saddr)
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
            if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            __syncwarp();
        }
    } else {
        const unsigned long long per = (groups + gridDim.x - 1) / gridDim.x;
        const unsigned long long lo = blockIdx.x * per;
        const unsigned long long hi = lo + per < groups ? lo + per : groups;
        for (unsigned long long g = lo + threadIdx.x; g < hi; g += (unsigned long long)blockDim.x * U)
            body<R, W, V, U>(p, g, blockDim.x, hi, acc);
    }
    if (W == 0 && acc == 1.2345) *p.sink = acc;
}

__global__ void fill(double* p, unsigned long long n, double salt) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x)
        p[i] = 1.0 + double(i % 1000003) * 1e-7 + salt;
}

template <int R, int W, int V, int U, int MODE>
void run(const std::vector<double*>& bufs, size_t n, int sms) {
    P<R, W> p;
    for (int i = 0; i < R; ++i) p.in[i] = bufs[i];
    for (int j = 0; j < W; ++j) p.out[j] = bufs[R + j];
    p.sink = bufs.back();
    const unsigned long long groups = n / V;
    auto k = stream_kernel<R, W, V, U, MODE>;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0);
    unsigned grid = (MODE == 1 || MODE == 3)
                        ? unsigned((groups + 256ull * U - 1) / (256ull * U))
                        : unsigned(sms * per_sm);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) k<<<grid, 256>>>(p, groups);
    const int reps = 20;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) k<<<grid, 256>>>(p, groups);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double s = ms * 1e-3 / reps;
    const double bytes = double(n) * 8 * (R + W);
    printf("{\"mix\": \"%dR:%dW\", \"V\": %d, \"U\": %d, \"mode\": %d, \"points\": %zu, "
           "\"ms\": %.4f, \"GBps\": %.1f, \"ctas_per_sm\": %d, \"err\": \"%s\"}\n",
           R, W, V, U, MODE, n, s * 1e3, bytes / s / 1e9, per_sm,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
}

template <int R, int W>
void sweep(const std::vector<double*>& bufs, size_t n, int sms) {
    run<R, W, 4, 1, 0>(bufs, n, sms);
    run<R, W, 4, 2, 0>(bufs, n, sms);
    run<R, W, 2, 2, 0>(bufs, n, sms);
    run<R, W, 4, 1, 1>(bufs, n, sms);
    run<R, W, 4, 2, 1>(bufs, n, sms);
    run<R, W, 4, 4, 1>(bufs, n, sms);
    run<R, W, 2, 4, 1>(bufs, n, sms);
    run<R, W, 4, 1, 2>(bufs, n, sms);
    run<R, W, 4, 2, 2>(bufs, n, sms);
    if constexpr (W > 0) run<R, W, 4, 1, 3>(bufs, n, sms);
}

int main(int argc, char** argv) {
    size_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 100000000ull;
    n &= ~size_t(15);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    std::vector<double*> bufs(21);
    for (int i = 0; i < 21; ++i) {
        if (cudaMalloc(&bufs[i], n * 8) != cudaSuccess) return 1;
        fill<<<sms * 8, 256>>>(bufs[i], n, i);
    }
    cudaDeviceSynchronize();
    sweep<1, 1>(bufs, n, sms);   // copy: the MEASURED_PEAKS denominator's mix
    sweep<5, 15>(bufs, n, sms);  // 3D flux
    sweep<3, 3>(bufs, n, sms);   // 1D cons->prim
    sweep<2, 1>(bufs, n, sms);   // axpy-sin
    sweep<5, 0>(bufs, n, sms);   // read-only CFL pass
    // 3-D Jacobians: 80 planes, at a quarter of N
    for (double* b : bufs) cudaFree(b);
    const size_t nj = (n / 4) & ~size_t(15);
    std::vector<double*> jb(81);
    for (int i = 0; i < 81; ++i) {
        if (cudaMalloc(&jb[i], nj * 8) != cudaSuccess) return 1;
        fill<<<sms * 8, 256>>>(jb[i], nj, i);
    }
    cudaDeviceSynchronize();
    run<5, 75, 4, 1, 1>(jb, nj, sms);
    run<5, 75, 4, 1, 3>(jb, nj, sms);
    run<5, 75, 4, 1, 0>(jb, nj, sms);
    return 0;
}
