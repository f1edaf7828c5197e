// fvb_sparse.cu -- the CSR block-matvec accumulation of the reference's
// block layer on the device (paper Eq. 2).
//
// proj/src/block.cpp:345-357 (csr_matvec_acc_t): for every row r,
//     acc = 0;  for k in row r (stored, column-sorted order):
//         acc += (TY)v[k] * (TY)x[ci[k]];
//     y[r] += acc;
// in the destination's precision TY.  The additions of one row must happen
// in stored order (that is the bitwise contract), but the products are
// independent: each is the same two roundings whichever thread computes it.
//
// So a warp owns 32 consecutive rows, whose nonzeros are one contiguous
// range of the CSR arrays.  The warp streams that range in tiles of
// kTile entries with coalesced loads (lane l takes entries l, l+32, ...),
// computes every product once and parks it in shared memory; then each lane
// adds up the products of its own row, in order, carrying acc from tile to
// tile.  Values and column indices -- 16 of the ~20 bytes per nonzero --
// are read as full 128-byte lines instead of one scattered word per row per
// thread, and the sum associates exactly as the reference's
// (--fmad=false keeps the multiply and the add separately rounded).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "fvb.h"
#include "fvb_dispatch.cuh"

namespace fvb {
namespace {

constexpr int kCsrThreads = 256;
constexpr int kTile = 256;  // products staged per warp per round

// Row per thread, nonzeros walked in stored order (the simple form; kept for
// the comparison in tools/csr_bench.py via FVB_CSR_MODE=row).
template <class TY, class TX, class IT>
__global__ void __launch_bounds__(kCsrThreads)
    csr_row_kernel(uint64_t rows, const uint64_t* __restrict__ rp, const IT* __restrict__ ci,
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

// Warp-staged: see the file comment.  One warp per 32 rows, grid-stride.
template <class TY, class TX, class IT, int MINB, int UNR>
__global__ void __launch_bounds__(kCsrThreads, MINB)
    csr_warp_kernel(uint64_t rows, const uint64_t* __restrict__ rp,
                    const IT* __restrict__ ci, const double* __restrict__ v,
                    const TX* __restrict__ x, TY* __restrict__ y) {
    __shared__ TY prod[kCsrThreads / 32][kTile];
    const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    TY* p = prod[wib];
    const uint64_t warps = uint64_t(gridDim.x) * (kCsrThreads / 32);
    for (uint64_t w = uint64_t(blockIdx.x) * (kCsrThreads / 32) + wib; w * 32 < rows; w += warps) {
        const uint64_t r = w * 32 + lane;
        const bool valid = r < rows;
        const uint64_t beg = valid ? rp[r] : 0;
        const uint64_t end = valid ? rp[r + 1] : 0;
        const uint64_t last = rows - w * 32 < 32 ? rows - w * 32 - 1 : 31;
        const uint64_t B = __shfl_sync(0xffffffffu, beg, 0);
        const uint64_t E = __shfl_sync(0xffffffffu, end, unsigned(last));
        TY acc = 0;
        for (uint64_t base = B; base < E; base += kTile) {
            const unsigned lim = E - base < uint64_t(kTile) ? unsigned(E - base) : unsigned(kTile);
            const double* vb = v + base;
            const IT* cb = ci + base;
#pragma unroll UNR
            for (unsigned t = lane; t < lim; t += 32)
                p[t] = static_cast<TY>(vb[t]) * static_cast<TY>(x[cb[t]]);
            __syncwarp();
            // this lane's row within the tile: [clamp(beg-base), clamp(end-base))
            const unsigned lo = beg <= base ? 0u : (beg - base < lim ? unsigned(beg - base) : lim);
            const unsigned hi = end <= base ? 0u : (end - base < lim ? unsigned(end - base) : lim);
            for (unsigned k = lo; k < hi; ++k) acc = acc + p[k];
            __syncwarp();
        }
        if (valid) y[r] = y[r] + acc;
    }
}

// FVB_CSR_MODE=row selects the row-per-thread form (FVB_CSR_ROWWISE=1 is the
// older spelling), FVB_CSR_MODE=warp the default; read per call so tests
// cover both in one process.  (A TMA bulk-copy ring was measured at 0.58 of
// peak at best and not adopted: profiles/r01_csr_shapes.txt, commit 2d1fa1d.)
bool rowwise() {
    const char* m = std::getenv("FVB_CSR_MODE");
    if (m && *m) return !std::strcmp(m, "row");
    const char* e = std::getenv("FVB_CSR_ROWWISE");
    return e && *e && *e != '0';
}

template <class TY, class TX, class IT>
fvb_status launch_csr(uint64_t rows, const uint64_t* rp, const IT* ci, const double* v,
                      const void* x, void* y, cudaStream_t s) {
    if (rowwise()) {
        csr_row_kernel<TY, TX, IT><<<simple_grid(rows), kCsrThreads, 0, s>>>(
            rows, rp, ci, v, static_cast<const TX*>(x), static_cast<TY*>(y));
    } else {
        // one pass over the rows: a warp per 32 rows, capped at a few waves
        const uint64_t warps = (rows + 31) / 32;
        uint64_t grid = (warps + kCsrThreads / 32 - 1) / (kCsrThreads / 32);
        const uint64_t cap = uint64_t(device_sm_count()) * 8 * 64;
        grid = grid < cap ? grid : cap;
        const unsigned g = unsigned(grid ? grid : 1);
        const TX* xx = static_cast<const TX*>(x);
        TY* yy = static_cast<TY*>(y);
        // 8 resident CTAs (32 registers) and three tile entries in flight
        // per lane: the measured best (profiles/r01_csr_shapes.txt)
        const char* u = std::getenv("FVB_CSR_UNROLL");  // sweep knob: 2, 3 (default), 4
        if (u && !std::strcmp(u, "4"))
            csr_warp_kernel<TY, TX, IT, 8, 4><<<g, kCsrThreads, 0, s>>>(rows, rp, ci, v, xx, yy);
        else if (u && !std::strcmp(u, "2"))
            csr_warp_kernel<TY, TX, IT, 8, 2><<<g, kCsrThreads, 0, s>>>(rows, rp, ci, v, xx, yy);
        else
            csr_warp_kernel<TY, TX, IT, 8, 3><<<g, kCsrThreads, 0, s>>>(rows, rp, ci, v, xx, yy);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FVB_OK : cuda_fail(e, "csr matvec launch");
}

template <class IT>
fvb_status csr_entry(uint8_t prec_y, uint8_t prec_x, uint64_t rows, uint64_t nnz,
                     const uint64_t* row_ptr, const IT* col_idx, const double* values,
                     const void* x, void* y, void* stream) {
    if (prec_y > 1 || prec_x > 1) return fail(FVB_EPREC, "precision code must be 0 or 1");
    if (rows == 0) return FVB_OK;
    if (!row_ptr || !y || (nnz && (!col_idx || !values || !x)))
        return fail(FVB_EARG, "NULL CSR array or plane");
    auto s = static_cast<cudaStream_t>(stream);
    if (prec_y == FVB_F64)
        return prec_x == FVB_F64
                   ? launch_csr<double, double, IT>(rows, row_ptr, col_idx, values, x, y, s)
                   : launch_csr<double, float, IT>(rows, row_ptr, col_idx, values, x, y, s);
    return prec_x == FVB_F64 ? launch_csr<float, double, IT>(rows, row_ptr, col_idx, values, x, y, s)
                             : launch_csr<float, float, IT>(rows, row_ptr, col_idx, values, x, y, s);
}

}  // namespace
}  // namespace fvb

using namespace fvb;

extern "C" {

fvb_status fvb_csr_matvec_acc(uint8_t prec_y, uint8_t prec_x, uint64_t rows, uint64_t nnz,
                              const uint64_t* row_ptr, const uint64_t* col_idx,
                              const double* values, const void* x, void* y, void* stream) {
    return csr_entry(prec_y, prec_x, rows, nnz, row_ptr, col_idx, values, x, y, stream);
}

fvb_status fvb_csr_matvec_acc_u32(uint8_t prec_y, uint8_t prec_x, uint64_t rows, uint64_t nnz,
                                  const uint64_t* row_ptr, const uint32_t* col_idx,
                                  const double* values, const void* x, void* y, void* stream) {
    return csr_entry(prec_y, prec_x, rows, nnz, row_ptr, col_idx, values, x, y, stream);
}

}  // extern "C"
