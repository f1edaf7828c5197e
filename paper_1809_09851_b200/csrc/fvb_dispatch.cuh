// fvb_dispatch.cuh -- argument checks and (dimension, precision) dispatch
// shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include "fvb.h"
#include "fvb_launch.cuh"

namespace fvb {

inline fvb_status check_common(uint32_t dim, uint8_t prec, bool need_dim = true) {
    if (prec > 1) return fail(FVB_EPREC, "precision code must be 0 (f32) or 1 (f64)");
    if (need_dim && (dim < 1 || dim > 3)) return fail(FVB_EARG, "dim must be 1, 2 or 3");
    return FVB_OK;
}

inline fvb_status check_gas(const fvb_gas* g) {
    if (!g) return FVB_OK;
    if (!(g->cv > 0) || !(g->gamma_minus_one > 0) || !(g->gamma > 1))
        return fail(FVB_EARG, "gas constants must satisfy cv > 0, gamma-1 > 0, gamma > 1");
    return FVB_OK;
}

// reset_red: the reduction word is zeroed (after validation) before the
// kernel accumulates into it.
template <template <class, int> class OpT, bool RED, bool TUNE3, class T>
fvb_status run_dim(uint32_t dim, const void* const* in, void* const* out, uint64_t n,
                   const fvb_gas* gas, typename Bits<T>::U* red, cudaStream_t s,
                   bool reset_red = false) {
    const auto k = make_consts<T>(gas);
    auto i = reinterpret_cast<const T* const*>(in);
    auto o = reinterpret_cast<T* const*>(out);
    switch (dim) {
        case 1: return launch_op<OpT<T, 1>, T, RED, false>(i, o, n, k, red, s, reset_red);
        case 2: return launch_op<OpT<T, 2>, T, RED, false>(i, o, n, k, red, s, reset_red);
        default: return launch_op<OpT<T, 3>, T, RED, TUNE3>(i, o, n, k, red, s, reset_red);
    }
}

template <class T, int D>
using WaveSpeed0 = WaveSpeedOp<T, D, 0>;
template <class T, int D>
using WaveSpeed1 = WaveSpeedOp<T, D, 1>;

unsigned simple_grid(uint64_t n);

}  // namespace fvb
