// fvb_flux.cu -- fvb_flux: the fused (d+2) x d inviscid-flux block
// (proj/src/fluid.cpp:273-310), the headline kernel.
#include <cuda_runtime.h>

#include "fvb.h"
#include "fvb_dispatch.cuh"

using namespace fvb;

extern "C" {

fvb_status fvb_flux(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                    const void* const* in, void* const* out, void* stream) {
    if (fvb_status st = check_common(dim, prec)) return st;
    if (fvb_status st = check_gas(gas)) return st;
    if (!in || !out) return fail(FVB_EARG, "NULL plane array");
    auto s = static_cast<cudaStream_t>(stream);
    if (prec == FVB_F64) return run_dim<FluxOp, false, true, double>(dim, in, out, n, gas, nullptr, s);
    return run_dim<FluxOp, false, true, float>(dim, in, out, n, gas, nullptr, s);
}

fvb_status fvb_flux_prim(const fvb_gas* gas, uint32_t dim, uint8_t prec, uint64_t n,
                         const void* const* in, void* const* out, void* stream) {
    if (fvb_status st = check_common(dim, prec)) return st;
    if (fvb_status st = check_gas(gas)) return st;
    if (!in || !out) return fail(FVB_EARG, "NULL plane array");
    auto s = static_cast<cudaStream_t>(stream);
    if (prec == FVB_F64)
        return run_dim<FluxPrimOp, false, false, double>(dim, in, out, n, gas, nullptr, s);
    return run_dim<FluxPrimOp, false, false, float>(dim, in, out, n, gas, nullptr, s);
}

}  // extern "C"
