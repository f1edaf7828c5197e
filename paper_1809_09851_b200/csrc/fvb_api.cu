// fvb_api.cu -- the C ABI of include/fvb.h: validation, dispatch over
// (dimension, precision) and launch of the fused kernels.  No exceptions
// cross the boundary; every failure is an fvb_status plus a thread-local
// message, validated before anything is enqueued (as the reference's
// validate() throws before evaluating: proj/src/backend_eval.cpp:236-265).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "fvb.h"
#include "fvb_launch.cuh"

namespace fvb {

namespace {
thread_local std::string t_error;
}

void set_error(const std::string& msg) { t_error = msg; }

fvb_status fail(fvb_status s, const std::string& msg) {
    t_error = msg;
    return s;
}

fvb_status cuda_fail(cudaError_t e, const char* what) {
    t_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return FVB_ECUDA;
}

int device_sm_count() {
    static int counts[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!counts[dev]) {
        int c = 0;
        if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || c < 1)
            c = 148;
        counts[dev] = c;
    }
    return counts[dev];
}

const Tuning& tuning() {
    static const Tuning t = [] {
        Tuning x;
        auto env = [](const char* name, int dflt) {
            const char* v = std::getenv(name);
            return v && *v ? std::atoi(v) : dflt;
        };
        x.vec = env("FVB_VEC", 0);
        x.unroll = env("FVB_UNROLL", 1);
        x.store = env("FVB_STORE", kStoreStreaming);
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

// ---- dispatch helpers ------------------------------------------------------------

fvb_status check_common(uint32_t dim, uint8_t prec, bool need_dim = true) {
    if (prec > 1) return fail(FVB_EPREC, "precision code must be 0 (f32) or 1 (f64)");
    if (need_dim && (dim < 1 || dim > 3)) return fail(FVB_EARG, "dim must be 1, 2 or 3");
    return FVB_OK;
}

fvb_status check_gas(const fvb_gas* g) {
    if (!g) return FVB_OK;
    if (!(g->cv > 0) || !(g->gamma_minus_one > 0) || !(g->gamma > 1))
        return fail(FVB_EARG, "gas constants must satisfy cv > 0, gamma-1 > 0, gamma > 1");
    return FVB_OK;
}

template <template <class, int> class OpT, bool RED, bool TUNE3, class T>
fvb_status run_dim(uint32_t dim, const void* const* in, void* const* out, uint64_t n,
                   const fvb_gas* gas, typename Bits<T>::U* red, cudaStream_t s) {
    const auto k = make_consts<T>(gas);
    auto i = reinterpret_cast<const T* const*>(in);
    auto o = reinterpret_cast<T* const*>(out);
    switch (dim) {
        case 1: return launch_op<OpT<T, 1>, T, RED, false>(i, o, n, k, red, s);
        case 2: return launch_op<OpT<T, 2>, T, RED, false>(i, o, n, k, red, s);
        default: return launch_op<OpT<T, 3>, T, RED, TUNE3>(i, o, n, k, red, s);
    }
}

template <class T, int D>
using WaveSpeed0 = WaveSpeedOp<T, D, 0>;
template <class T, int D>
using WaveSpeed1 = WaveSpeedOp<T, D, 1>;

// Reset the device scalar, then let the kernel atomic-max into it (all in
// stream order, so concurrent calls on different outputs never interfere).
template <class T>
fvb_status reset_scalar(void* p, cudaStream_t s) {
    const cudaError_t e = cudaMemsetAsync(p, 0, sizeof(T), s);
    return e == cudaSuccess ? FVB_OK : cuda_fail(e, "lambda_max reset");
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

fvb_status fvb_axpy_sin(uint8_t prec, uint64_t n, const void* x, void* y, void* stream) {
    if (fvb_status st = check_common(1, prec, false)) return st;
    if (n == 0) return FVB_OK;
    if (!x || !y) return fail(FVB_EARG, "NULL plane");
    auto s = static_cast<cudaStream_t>(stream);
    if (prec == FVB_F64) {
        const double* in[2] = {static_cast<const double*>(x), static_cast<const double*>(y)};
        double* out[1] = {static_cast<double*>(y)};
        return launch_op<AxpySinOp<double>, double, false, false>(in, out, n, make_consts<double>(nullptr), nullptr, s);
    }
    const float* in[2] = {static_cast<const float*>(x), static_cast<const float*>(y)};
    float* out[1] = {static_cast<float*>(y)};
    return launch_op<AxpySinOp<float>, float, false, false>(in, out, n, make_consts<float>(nullptr), nullptr, s);
}

fvb_status fvb_flux(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                    const void* const* in, void* const* out, void* stream) {
    if (fvb_status st = check_common(dim, prec)) return st;
    if (fvb_status st = check_gas(gas)) return st;
    if (!in || !out) return fail(FVB_EARG, "NULL plane array");
    auto s = static_cast<cudaStream_t>(stream);
    if (prec == FVB_F64) return run_dim<FluxOp, false, true, double>(dim, in, out, n, gas, nullptr, s);
    return run_dim<FluxOp, false, true, float>(dim, in, out, n, gas, nullptr, s);
}

fvb_status fvb_cons2prim(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                         const void* const* in, void* const* out, void* stream) {
    if (fvb_status st = check_common(dim, prec)) return st;
    if (fvb_status st = check_gas(gas)) return st;
    if (!in || !out) return fail(FVB_EARG, "NULL plane array");
    auto s = static_cast<cudaStream_t>(stream);
    if (prec == FVB_F64)
        return run_dim<Cons2PrimOp, false, false, double>(dim, in, out, n, gas, nullptr, s);
    return run_dim<Cons2PrimOp, false, false, float>(dim, in, out, n, gas, nullptr, s);
}

fvb_status fvb_prim2cons(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                         const void* const* in, void* const* out, void* stream) {
    if (fvb_status st = check_common(dim, prec)) return st;
    if (fvb_status st = check_gas(gas)) return st;
    if (!in || !out) return fail(FVB_EARG, "NULL plane array");
    auto s = static_cast<cudaStream_t>(stream);
    if (prec == FVB_F64)
        return run_dim<Prim2ConsOp, false, false, double>(dim, in, out, n, gas, nullptr, s);
    return run_dim<Prim2ConsOp, false, false, float>(dim, in, out, n, gas, nullptr, s);
}

fvb_status fvb_v_mag2(uint32_t dim, uint8_t prec, uint64_t n, const void* const* in, void* out,
                      void* stream) {
    if (fvb_status st = check_common(dim, prec)) return st;
    if (!in || !out) return fail(FVB_EARG, "NULL plane");
    auto s = static_cast<cudaStream_t>(stream);
    void* const outs[1] = {out};
    if (prec == FVB_F64)
        return run_dim<VMag2Op, false, false, double>(dim, in, outs, n, nullptr, nullptr, s);
    return run_dim<VMag2Op, false, false, float>(dim, in, outs, n, nullptr, nullptr, s);
}

fvb_status fvb_eos(const fvb_gas* gas, uint8_t prec, uint64_t n, const void* rho, const void* e,
                   void* p, void* T, void* stream) {
    if (fvb_status st = check_common(1, prec, false)) return st;
    if (fvb_status st = check_gas(gas)) return st;
    if (n == 0 || (!p && !T)) return FVB_OK;
    if (!rho || !e) return fail(FVB_EARG, "NULL input plane");
    auto s = static_cast<cudaStream_t>(stream);
    auto go = [&](auto tag) -> fvb_status {
        using R = decltype(tag);
        const auto k = make_consts<R>(gas);
        const R* in[2] = {static_cast<const R*>(rho), static_cast<const R*>(e)};
        if (p && T) {
            R* out[2] = {static_cast<R*>(p), static_cast<R*>(T)};
            return launch_op<EosOp<R, 3>, R, false, false>(in, out, n, k, nullptr, s);
        }
        if (p) {
            R* out[1] = {static_cast<R*>(p)};
            return launch_op<EosOp<R, 1>, R, false, false>(in, out, n, k, nullptr, s);
        }
        R* out[1] = {static_cast<R*>(T)};
        return launch_op<EosOp<R, 2>, R, false, false>(in, out, n, k, nullptr, s);
    };
    return prec == FVB_F64 ? go(double(0)) : go(float(0));
}

fvb_status fvb_jacobian(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                        const void* const* in, void* const* out, void* lambda_max,
                        void* stream) {
    if (fvb_status st = check_common(dim, prec)) return st;
    if (fvb_status st = check_gas(gas)) return st;
    if (!in || !out) return fail(FVB_EARG, "NULL plane array");
    auto s = static_cast<cudaStream_t>(stream);
    if (prec == FVB_F64) {
        if (!lambda_max)
            return run_dim<JacobianOp, false, false, double>(dim, in, out, n, gas, nullptr, s);
        if (fvb_status st = reset_scalar<double>(lambda_max, s)) return st;
        return run_dim<JacobianOp, true, false, double>(
            dim, in, out, n, gas, static_cast<unsigned long long*>(lambda_max), s);
    }
    if (!lambda_max)
        return run_dim<JacobianOp, false, false, float>(dim, in, out, n, gas, nullptr, s);
    if (fvb_status st = reset_scalar<float>(lambda_max, s)) return st;
    return run_dim<JacobianOp, true, false, float>(dim, in, out, n, gas,
                                                  static_cast<unsigned int*>(lambda_max), s);
}

fvb_status fvb_wave_speed_max(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                              const void* const* in, void* lambda, void* lambda_max,
                              void* stream) {
    if (fvb_status st = check_common(dim, prec)) return st;
    if (fvb_status st = check_gas(gas)) return st;
    if (!in) return fail(FVB_EARG, "NULL plane array");
    if (!lambda_max) return fail(FVB_EARG, "lambda_max must be a device scalar");
    auto s = static_cast<cudaStream_t>(stream);
    void* const outs[1] = {lambda};
    if (prec == FVB_F64) {
        if (fvb_status st = reset_scalar<double>(lambda_max, s)) return st;
        auto red = static_cast<unsigned long long*>(lambda_max);
        if (lambda) return run_dim<WaveSpeed1, true, false, double>(dim, in, outs, n, gas, red, s);
        return run_dim<WaveSpeed0, true, false, double>(dim, in, outs, n, gas, red, s);
    }
    if (fvb_status st = reset_scalar<float>(lambda_max, s)) return st;
    auto red = static_cast<unsigned int*>(lambda_max);
    if (lambda) return run_dim<WaveSpeed1, true, false, float>(dim, in, outs, n, gas, red, s);
    return run_dim<WaveSpeed0, true, false, float>(dim, in, outs, n, gas, red, s);
}

fvb_status fvb_synth_state(uint32_t dim, uint8_t prec, uint64_t seed, uint64_t first, uint64_t n,
                           void* const* out, void* stream) {
    if (fvb_status st = check_common(dim, prec)) return st;
    if (n == 0) return FVB_OK;
    if (!out) return fail(FVB_EARG, "NULL plane array");
    for (uint32_t i = 0; i < dim + 2; ++i)
        if (!out[i]) return fail(FVB_EARG, "NULL output plane");
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
