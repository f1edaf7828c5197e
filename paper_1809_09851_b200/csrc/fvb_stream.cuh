// fvb_stream.cuh -- wide streaming loads/stores and the generic fused
// pointwise kernel every block expression runs through.
//
// Memory model: SoA planes, one coalesced stream per
// plane.  A thread moves V consecutive elements of every plane per access:
// V*sizeof(T) = 32 bytes for the default V (sm_100's 256-bit LDG/STG,
// `LDG.E.*.256` / `STG.E.*.256` in SASS), so a warp touches one contiguous
// 1 KiB span per plane per access.  Inputs are read once through the
// non-coherent path without L1 allocation; outputs are written with an
// evict-first policy so the ~12 GB of flux output streaming through the
// 126 MB L2 does not evict lines still being read.
#pragma once

#include <cstdint>

#include "fvb_ops.cuh"

namespace fvb {

enum StorePolicy : int {
    kStoreDefault = 0,  // st.global
    kStoreStreaming = 1,  // st.global.cs   (evict-first)
    kStoreNoAlloc = 2,  // st.global.L1::no_allocate
};

// ---- loads ----------------------------------------------------------------

template <class T, int V>
struct VecIO;

template <>
struct VecIO<double, 1> {
    template <bool NC = true>
    __device__ __forceinline__ static void load(const double* p, double (&x)[1]) {
        if (NC)
            asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(x[0]) : "l"(p));
        else
            asm volatile("ld.global.f64 %0, [%1];" : "=d"(x[0]) : "l"(p) : "memory");
    }
    template <int SP>
    __device__ __forceinline__ static void store(double* p, const double (&x)[1]) {
        if (SP == kStoreStreaming)
            asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(x[0]) : "memory");
        else if (SP == kStoreNoAlloc)
            asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(x[0]) : "memory");
        else
            asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(x[0]) : "memory");
    }
};

template <>
struct VecIO<double, 2> {
    template <bool NC = true>
    __device__ __forceinline__ static void load(const double* p, double (&x)[2]) {
        if (NC)
            asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                         : "=d"(x[0]), "=d"(x[1])
                         : "l"(p));
        else
            asm volatile("ld.global.v2.f64 {%0, %1}, [%2];"
                         : "=d"(x[0]), "=d"(x[1])
                         : "l"(p)
                         : "memory");
    }
    template <int SP>
    __device__ __forceinline__ static void store(double* p, const double (&x)[2]) {
        if (SP == kStoreStreaming)
            asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(x[0]), "d"(x[1])
                         : "memory");
        else if (SP == kStoreNoAlloc)
            asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(x[0]),
                         "d"(x[1])
                         : "memory");
        else
            asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(x[0]), "d"(x[1])
                         : "memory");
    }
};

template <>
struct VecIO<double, 4> {
    template <bool NC = true>
    __device__ __forceinline__ static void load(const double* p, double (&x)[4]) {
        if (NC)
            asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
                         : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
                         : "l"(p));
        else
            asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                         : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
                         : "l"(p)
                         : "memory");
    }
    template <int SP>
    __device__ __forceinline__ static void store(double* p, const double (&x)[4]) {
        if (SP == kStoreStreaming)
            asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(x[0]),
                         "d"(x[1]), "d"(x[2]), "d"(x[3])
                         : "memory");
        else if (SP == kStoreNoAlloc)
            asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p),
                         "d"(x[0]), "d"(x[1]), "d"(x[2]), "d"(x[3])
                         : "memory");
        else
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(x[0]),
                         "d"(x[1]), "d"(x[2]), "d"(x[3])
                         : "memory");
    }
};

template <>
struct VecIO<float, 1> {
    template <bool NC = true>
    __device__ __forceinline__ static void load(const float* p, float (&x)[1]) {
        if (NC)
            asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(x[0]) : "l"(p));
        else
            asm volatile("ld.global.f32 %0, [%1];" : "=f"(x[0]) : "l"(p) : "memory");
    }
    template <int SP>
    __device__ __forceinline__ static void store(float* p, const float (&x)[1]) {
        if (SP == kStoreStreaming)
            asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(x[0]) : "memory");
        else if (SP == kStoreNoAlloc)
            asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(p), "f"(x[0]) : "memory");
        else
            asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(x[0]) : "memory");
    }
};

template <>
struct VecIO<float, 4> {
    template <bool NC = true>
    __device__ __forceinline__ static void load(const float* p, float (&x)[4]) {
        if (NC)
            asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3])
                         : "l"(p));
        else
            asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3])
                         : "l"(p)
                         : "memory");
    }
    template <int SP>
    __device__ __forceinline__ static void store(float* p, const float (&x)[4]) {
        if (SP == kStoreStreaming)
            asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(x[0]),
                         "f"(x[1]), "f"(x[2]), "f"(x[3])
                         : "memory");
        else if (SP == kStoreNoAlloc)
            asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                         "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3])
                         : "memory");
        else
            asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(x[0]),
                         "f"(x[1]), "f"(x[2]), "f"(x[3])
                         : "memory");
    }
};

template <>
struct VecIO<float, 8> {
    template <bool NC = true>
    __device__ __forceinline__ static void load(const float* p, float (&x)[8]) {
        if (NC)
            asm volatile(
                "ld.global.nc.L1::no_allocate.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]),
                  "=f"(x[6]), "=f"(x[7])
                : "l"(p));
        else
            asm volatile("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]),
                           "=f"(x[5]), "=f"(x[6]), "=f"(x[7])
                         : "l"(p)
                         : "memory");
    }
    template <int SP>
    __device__ __forceinline__ static void store(float* p, const float (&x)[8]) {
        if (SP == kStoreStreaming)
            asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p),
                         "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]), "f"(x[4]), "f"(x[5]),
                         "f"(x[6]), "f"(x[7])
                         : "memory");
        else if (SP == kStoreNoAlloc)
            asm volatile(
                "st.global.L1::no_allocate.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(
                    p),
                "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]),
                "f"(x[7])
                : "memory");
        else
            asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p),
                         "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]), "f"(x[4]), "f"(x[5]),
                         "f"(x[6]), "f"(x[7])
                         : "memory");
    }
};

// ---- max-reduction helpers (lambda >= 0 or NaN) ----------------------------
// For non-negative IEEE values the unsigned bit pattern orders like the value,
// and every NaN pattern (sign set or not) sorts above +inf, so an unsigned
// max both finds the maximum exactly and propagates NaN.  The result is
// order-independent, hence bitwise invariant to grid shape and GPU count.

template <class T>
struct Bits;
template <>
struct Bits<double> {
    using U = unsigned long long;
    __device__ __forceinline__ static U of(double x) {
        return static_cast<U>(__double_as_longlong(x));
    }
};
template <>
struct Bits<float> {
    using U = unsigned int;
    __device__ __forceinline__ static U of(float x) { return __float_as_uint(x); }
};

template <class U>
__device__ __forceinline__ U warp_max_u(U v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        U o = __shfl_xor_sync(0xffffffffu, v, off);
        v = o > v ? o : v;
    }
    return v;
}

// ---- the fused pointwise kernel ---------------------------------------------

template <class T, int NIN, int NOUT>
struct Planes {
    const T* in[NIN];
    T* out[NOUT > 0 ? NOUT : 1];
};

// Index space: [0, head) scalar, then `groups` vector groups of V elements
// starting at `head`, then `tail` scalar elements.  head aligns every plane
// to V*sizeof(T) bytes (the host checks all planes share one residue).
struct Range {
    uint64_t head;
    uint64_t groups;
    uint64_t tail;
};

template <class Op, class T>
__device__ __forceinline__ void point_scalar(const Planes<T, Op::NIN, Op::NOUT>& pl,
                                             const Consts<T>& k, uint64_t idx,
                                             typename Bits<T>::U& acc) {
    T in[Op::NIN];
#pragma unroll
    for (int i = 0; i < Op::NIN; ++i) {
        T x[1];
        VecIO<T, 1>::template load<!Op::ALIASED>(pl.in[i] + idx, x);
        in[i] = x[0];
    }
    const typename Op::State s = Op::prepare(in, k);
#pragma unroll
    for (int j = 0; j < Op::NOUT; ++j) {
        T o[1] = {Op::out(s, j, k)};
        VecIO<T, 1>::template store<kStoreDefault>(pl.out[j] + idx, o);
    }
    if (Op::HAS_LAMBDA) {
        const auto b = Bits<T>::of(Op::lambda(s, k));
        acc = b > acc ? b : acc;
    }
}

// One trip of a thread: U groups (g0, g0+step, ...) -- all U*NIN wide loads
// issued first, then the per-point arithmetic and the NOUT wide stores.
template <class Op, class T, int V, int U, int SP, bool REDUCE>
__device__ __forceinline__ void pointwise_trip(const Planes<T, Op::NIN, Op::NOUT>& pl,
                                               const Consts<T>& k, const Range& rg, uint64_t g0,
                                               uint64_t step, typename Bits<T>::U& acc) {
    using Bu = typename Bits<T>::U;
    T x[U][Op::NIN][V];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t g = g0 + u * step;
        if (g < rg.groups) {
            const uint64_t base = rg.head + g * V;
#pragma unroll
            for (int i = 0; i < Op::NIN; ++i)
                VecIO<T, V>::template load<!Op::ALIASED>(pl.in[i] + base, x[u][i]);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t g = g0 + u * step;
        if (g < rg.groups) {
            const uint64_t base = rg.head + g * V;
            typename Op::State s[V];
#pragma unroll
            for (int q = 0; q < V; ++q) {
                T in[Op::NIN];
#pragma unroll
                for (int i = 0; i < Op::NIN; ++i) in[i] = x[u][i][q];
                s[q] = Op::prepare(in, k);
            }
#pragma unroll
            for (int j = 0; j < Op::NOUT; ++j) {
                T o[V];
#pragma unroll
                for (int q = 0; q < V; ++q) o[q] = Op::out(s[q], j, k);
                VecIO<T, V>::template store<SP>(pl.out[j] + base, o);
            }
            if (REDUCE) {
#pragma unroll
                for (int q = 0; q < V; ++q) {
                    const Bu b = Bits<T>::of(Op::lambda(s[q], k));
                    acc = b > acc ? b : acc;
                }
            }
        }
    }
}

// Launch shapes (template MODE), chosen by measurement (tools/hbm_probe.cu,
// DESIGN.md §Kernels):
//   kTiles      (default) one-shot grid; CTA b owns the U*THREADS consecutive
//               groups [b*U*THREADS, (b+1)*U*THREADS), thread t takes groups
//               t, t+THREADS, ...  Retiring CTAs are replaced by the block
//               scheduler, which spreads the streams over HBM; measured
//               +14% over a persistent sweep for every read/write mix.
//   kPersistent grid = SMs x resident CTAs, grid-stride over all groups.
enum LaunchMode : int { kPersistent = 0, kTiles = 1 };

// REDUCE: fold the CTA's lambda bits into *red with one atomicMax, skipped
// when a coherent read shows *red already at least as large (the running
// maximum rarely grows, so almost every CTA of a one-shot grid skips the
// atomic and a single address never becomes a serialisation point).
template <class Op, class T, int V, int U, int SP, bool REDUCE, int THREADS = 256, int MINB = 1,
          int MODE = kTiles>
__global__ void __launch_bounds__(THREADS, MINB)
    pointwise_kernel(const Planes<T, Op::NIN, Op::NOUT> pl, const Consts<T> k, const Range rg,
                     typename Bits<T>::U* __restrict__ red) {
    using Bu = typename Bits<T>::U;
    // Programmatic dependent launch (launch_fixed): this grid may have been
    // scheduled while the previous one on the stream was still draining.
    // Wait for it to complete (its memory visible) before touching any
    // plane; a no-op for an ordinary launch.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    Bu acc = 0;
    if (MODE == kTiles) {
        const uint64_t g0 = uint64_t(blockIdx.x) * (uint64_t(THREADS) * U) + threadIdx.x;
        pointwise_trip<Op, T, V, U, SP, REDUCE>(pl, k, rg, g0, THREADS, acc);
    } else {
        const uint64_t nthreads = uint64_t(gridDim.x) * THREADS;
        for (uint64_t g0 = uint64_t(blockIdx.x) * THREADS + threadIdx.x; g0 < rg.groups;
             g0 += nthreads * U)
            pointwise_trip<Op, T, V, U, SP, REDUCE>(pl, k, rg, g0, nthreads, acc);
    }

    // Unaligned head and ragged tail: at most 2V-2 elements, one per thread
    // of block 0.
    if (blockIdx.x == 0 && threadIdx.x < rg.head + rg.tail) {
        const uint64_t t = threadIdx.x;
        const uint64_t idx = t < rg.head ? t : rg.head + rg.groups * V + (t - rg.head);
        point_scalar<Op, T>(pl, k, idx, acc);
    }

    if (REDUCE) {
        __shared__ Bu warp_best[THREADS / 32];
        acc = warp_max_u(acc);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) warp_best[warp] = acc;
        __syncthreads();
        if (warp == 0) {
            Bu v = lane < THREADS / 32 ? warp_best[lane] : Bu(0);
            v = warp_max_u(v);
            if (lane == 0 && v != 0) {
                const Bu seen = *reinterpret_cast<volatile Bu*>(red);
                if (v > seen) atomicMax(red, v);
            }
        }
    }
    // This CTA's work is issued: the next grid may begin launching (it
    // still waits for this whole grid in its griddepcontrol.wait).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace fvb
