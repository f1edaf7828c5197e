// fvb_api.cu -- the C ABI of include/fvb.h: library entry points, error
// state, launch tuning and the on-device synthetic-input generators.  The
// fused blocks live in fvb_flux.cu, fvb_fluid.cu and fvb_jacobian.cu.  No exceptions
// cross the boundary; every failure is an fvb_status plus a thread-local
// message, validated before anything is enqueued (as the reference's
// validate() throws before evaluating: proj/src/backend_eval.cpp:236-265).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "fvb.h"
#include "fvb_dispatch.cuh"

namespace fvb {

namespace {
thread_local std::string t_error;
}

fvb_status fail(fvb_status s, const std::string& msg) {
    try {
        t_error = msg;
    } catch (...) {  // keep the status; the message is best effort
    }
    return s;
}

fvb_status cuda_fail(cudaError_t e, const char* what) {
    try {
        t_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    } catch (...) {
    }
    return FVB_ECUDA;
}

int device_sm_count() {
    static std::atomic<int> counts[64];  // 0 = not queried yet
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    int c = counts[dev].load(std::memory_order_relaxed);
    if (!c) {
        if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || c < 1)
            c = 148;
        counts[dev].store(c, std::memory_order_relaxed);
    }
    return c;
}

const Tuning& tuning() {
    static const Tuning t = [] {
        Tuning x;
        auto env = [](const char* name, int dflt) {
            const char* v = std::getenv(name);
            return v && *v ? std::atoi(v) : dflt;
        };
        x.vec = env("FVB_VEC", 0);
        x.unroll = env("FVB_UNROLL", 0);
        x.threads = env("FVB_THREADS", 0);
        x.min_blocks = env("FVB_MINB", 0);
        x.mode = env("FVB_MODE", 0);
        x.ctas_per_sm = env("FVB_CTAS", 0);
        return x;
    }();
    return t;
}

// ---- synthetic inputs --------------------------------------------------------

// SplitMix64 draw k of a generator seeded with `seed`
// (proj/include/fusevec/rng.hpp:12-18; state after k+1 calls).
__device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t k) {
    uint64_t z = seed + (k + 1ull) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// rng.uniform(lo, hi) (rng.hpp:21-23); exact IEEE ops under --fmad=false.
__device__ __forceinline__ double uniform_draw(uint64_t seed, uint64_t k, double lo, double hi) {
    const double u = double(splitmix_draw(seed, k) >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
}

template <class T, int D>
__global__ void __launch_bounds__(256)
    synth_state_kernel(uint64_t seed, uint64_t first, uint64_t n, Planes<T, 0 + 1, D + 2> pl) {
    // random_state of proj/tests/acceptance.cpp:214-230 for global point
    // first+t: draws rho, p, v_0..v_{d-1}; m_j = rho*v_j;
    // rhoE = p/0.4 + 0.5*rho*vsq (vsq accumulated from 0).
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += stride) {
        const uint64_t k0 = (first + t) * uint64_t(D + 2);
        const double rho = uniform_draw(seed, k0, 0.5, 2.0);
        const double p = uniform_draw(seed, k0 + 1, 0.5, 2.0);
        double vsq = 0;
        pl.out[0][t] = static_cast<T>(rho);
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const double v = uniform_draw(seed, k0 + 2 + j, -1.0, 1.0);
            vsq += v * v;
            pl.out[1 + j][t] = static_cast<T>(rho * v);
        }
        pl.out[D + 1][t] = static_cast<T>(p / 0.4 + 0.5 * rho * vsq);
    }
}

template <class T>
__global__ void __launch_bounds__(256)
    synth_uniform_kernel(uint64_t seed, uint64_t first, uint64_t n, double lo, double hi, T* out) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += stride)
        out[t] = static_cast<T>(uniform_draw(seed, first + t, lo, hi));
}

unsigned simple_grid(uint64_t n) {
    const uint64_t want = (n + 255) / 256;
    const uint64_t cap = uint64_t(device_sm_count()) * 8;
    return unsigned(want < cap ? (want ? want : 1) : cap);
}

}  // namespace fvb

using namespace fvb;

extern "C" {

int fvb_abi_version(void) { return FVB_ABI_VERSION; }

const char* fvb_last_error(void) { return t_error.c_str(); }

const char* fvb_build_info(void) {
    return "libfvb: sm_100a (compute_100a), --fmad=false, IEEE div/sqrt, 256-bit SoA streaming, "
           "nvcc " FVB_NVCC_VERSION;
}

fvb_status fvb_synth_state(uint32_t dim, uint8_t prec, uint64_t seed, uint64_t first, uint64_t n,
                           void* const* out, void* stream) {
    if (fvb_status st = check_common(dim, prec)) return st;
    if (n == 0) return FVB_OK;
    if (!out) return fail(FVB_EARG, "NULL plane array");
    const size_t w = prec == FVB_F64 ? 8 : 4;
    for (uint32_t i = 0; i < dim + 2; ++i) {
        if (!out[i]) return fail(FVB_EARG, "NULL output plane");
        // a misaligned store would be a sticky device fault, not an error code
        if (reinterpret_cast<uintptr_t>(out[i]) % w)
            return fail(FVB_EALIGN, "output plane is not element-aligned");
    }
    auto s = static_cast<cudaStream_t>(stream);
    const unsigned grid = simple_grid(n);
    auto go = [&](auto tag, auto dtag) {
        using R = decltype(tag);
        constexpr int D = decltype(dtag)::value;
        Planes<R, 1, D + 2> pl;
        pl.in[0] = nullptr;
        for (int i = 0; i < D + 2; ++i) pl.out[i] = static_cast<R*>(out[i]);
        synth_state_kernel<R, D><<<grid, 256, 0, s>>>(seed, first, n, pl);
    };
    if (prec == FVB_F64) {
        if (dim == 1) go(double(0), std::integral_constant<int, 1>());
        else if (dim == 2) go(double(0), std::integral_constant<int, 2>());
        else go(double(0), std::integral_constant<int, 3>());
    } else {
        if (dim == 1) go(float(0), std::integral_constant<int, 1>());
        else if (dim == 2) go(float(0), std::integral_constant<int, 2>());
        else go(float(0), std::integral_constant<int, 3>());
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FVB_OK : cuda_fail(e, "synth_state launch");
}

fvb_status fvb_synth_uniform(uint8_t prec, uint64_t seed, uint64_t first, uint64_t n, double lo,
                             double hi, void* out, void* stream) {
    if (fvb_status st = check_common(1, prec, false)) return st;
    if (n == 0) return FVB_OK;
    if (!out) return fail(FVB_EARG, "NULL plane");
    if (reinterpret_cast<uintptr_t>(out) % (prec == FVB_F64 ? 8 : 4))
        return fail(FVB_EALIGN, "output plane is not element-aligned");
    auto s = static_cast<cudaStream_t>(stream);
    if (prec == FVB_F64)
        synth_uniform_kernel<double><<<simple_grid(n), 256, 0, s>>>(seed, first, n, lo, hi,
                                                                    static_cast<double*>(out));
    else
        synth_uniform_kernel<float><<<simple_grid(n), 256, 0, s>>>(seed, first, n, lo, hi,
                                                                   static_cast<float*>(out));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FVB_OK : cuda_fail(e, "synth_uniform launch");
}

}  // extern "C"
