// fvb_sparse.cu -- the CSR block-matvec accumulation of the reference's
// block layer on the device (paper Eq. 2).
//
// proj/src/block.cpp:345-357 (csr_matvec_acc_t): for every row r,
//     acc = 0;  for k in row r (stored, column-sorted order):
//         acc += (TY)v[k] * (TY)x[ci[k]];
//     y[r] += acc;
// in the destination's precision TY.  One thread owns one row and walks its
// nonzeros in stored order, so the sum associates exactly as the reference's
// does and the result is bitwise identical (--fmad=false keeps the multiply
// and the add separately rounded).  Row-parallel, not nonzero-parallel: the
// reference's block matrices are short-row (PDE stencils); the order of the
// additions is the contract.
#include <cuda_runtime.h>

#include <cstdint>

#include "fvb.h"
#include "fvb_dispatch.cuh"

namespace fvb {
namespace {

template <class TY, class TX>
__global__ void __launch_bounds__(256)
    csr_acc_kernel(uint64_t rows, const uint64_t* __restrict__ rp, const uint64_t* __restrict__ ci,
                   const double* __restrict__ v, const TX* __restrict__ x, TY* __restrict__ y) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += stride) {
        TY acc = 0;
        const uint64_t end = rp[r + 1];
        for (uint64_t k = rp[r]; k < end; ++k)
            acc = acc + static_cast<TY>(v[k]) * static_cast<TY>(x[ci[k]]);
        y[r] = y[r] + acc;
    }
}

template <class TY, class TX>
fvb_status launch_csr(uint64_t rows, const uint64_t* rp, const uint64_t* ci, const double* v,
                      const void* x, void* y, cudaStream_t s) {
    csr_acc_kernel<TY, TX><<<simple_grid(rows), 256, 0, s>>>(
        rows, rp, ci, v, static_cast<const TX*>(x), static_cast<TY*>(y));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FVB_OK : cuda_fail(e, "csr matvec launch");
}

}  // namespace
}  // namespace fvb

using namespace fvb;

extern "C" {

fvb_status fvb_csr_matvec_acc(uint8_t prec_y, uint8_t prec_x, uint64_t rows, uint64_t nnz,
                              const uint64_t* row_ptr, const uint64_t* col_idx,
                              const double* values, const void* x, void* y, void* stream) {
    if (prec_y > 1 || prec_x > 1) return fail(FVB_EPREC, "precision code must be 0 or 1");
    if (rows == 0) return FVB_OK;
    if (!row_ptr || !y || (nnz && (!col_idx || !values || !x)))
        return fail(FVB_EARG, "NULL CSR array or plane");
    auto s = static_cast<cudaStream_t>(stream);
    if (prec_y == FVB_F64)
        return prec_x == FVB_F64 ? launch_csr<double, double>(rows, row_ptr, col_idx, values, x, y, s)
                                 : launch_csr<double, float>(rows, row_ptr, col_idx, values, x, y, s);
    return prec_x == FVB_F64 ? launch_csr<float, double>(rows, row_ptr, col_idx, values, x, y, s)
                             : launch_csr<float, float>(rows, row_ptr, col_idx, values, x, y, s);
}

}  // extern "C"
