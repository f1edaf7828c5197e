// fvb_jacobian.cu -- flux Jacobians fused with the CFL wave-speed maximum,
// and the read-only CFL pass.
#include <cuda_runtime.h>

#include "fvb.h"
#include "fvb_dispatch.cuh"

namespace fvb {
template <class T, int D>
using WaveSpeed0 = WaveSpeedOp<T, D, 0>;
template <class T, int D>
using WaveSpeed1 = WaveSpeedOp<T, D, 1>;
}  // namespace fvb

using namespace fvb;

extern "C" {

// The CFL word is zeroed in stream order (so concurrent calls on different
// words never interfere) by launch_op, once the planes have been validated.
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
        return run_dim<JacobianOp, true, false, double>(
            dim, in, out, n, gas, static_cast<unsigned long long*>(lambda_max), s, true);
    }
    if (!lambda_max)
        return run_dim<JacobianOp, false, false, float>(dim, in, out, n, gas, nullptr, s);
    return run_dim<JacobianOp, true, false, float>(dim, in, out, n, gas,
                                                  static_cast<unsigned int*>(lambda_max), s, true);
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
        auto red = static_cast<unsigned long long*>(lambda_max);
        if (lambda)
            return run_dim<WaveSpeed1, true, false, double>(dim, in, outs, n, gas, red, s, true);
        return run_dim<WaveSpeed0, true, true, double>(dim, in, outs, n, gas, red, s, true);
    }
    auto red = static_cast<unsigned int*>(lambda_max);
    if (lambda) return run_dim<WaveSpeed1, true, false, float>(dim, in, outs, n, gas, red, s, true);
    return run_dim<WaveSpeed0, true, true, float>(dim, in, outs, n, gas, red, s, true);
}

}  // extern "C"
