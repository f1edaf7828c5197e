// fvb_fluid.cu -- the remaining fused fluid blocks and the UETLI axpy-sin:
// cons->prim + EOS + sound speed, prim->cons, v_mag2, EOS closures.
#include <cuda_runtime.h>

#include "fvb.h"
#include "fvb_dispatch.cuh"

using namespace fvb;

extern "C" {

fvb_status fvb_axpy_sin(uint8_t prec, uint64_t n, const void* x, void* y, void* stream) {
    if (fvb_status st = check_common(1, prec, false)) return st;
    if (n == 0) return FVB_OK;
    if (!x || !y) return fail(FVB_EARG, "NULL plane");
    auto s = static_cast<cudaStream_t>(stream);
    if (prec == FVB_F64) {
        const double* in[2] = {static_cast<const double*>(x), static_cast<const double*>(y)};
        double* out[1] = {static_cast<double*>(y)};
        return launch_op<AxpySinOp<double>, double, false, true>(in, out, n, make_consts<double>(nullptr), nullptr, s);
    }
    const float* in[2] = {static_cast<const float*>(x), static_cast<const float*>(y)};
    float* out[1] = {static_cast<float*>(y)};
    return launch_op<AxpySinOp<float>, float, false, true>(in, out, n, make_consts<float>(nullptr), nullptr, s);
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
    if (n == 0) return FVB_OK;
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

}  // extern "C"
