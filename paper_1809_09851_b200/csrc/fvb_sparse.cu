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

// ---- the asynchronous pipeline form (FVB_CSR_MODE=pipe) -----------------------
//
// The warp-staged form holds every in-flight load in registers, so memory
// parallelism per SM is capped by the register file: a unit of 32 rows
// walks rp -> (v, ci) -> x -> y, about eight dependent round trips, and 64
// warps per SM keep ~8 units in flight.  Here every load is a cp.async
// (LDGSTS) into the warp's shared memory -- no register holds in-flight
// data -- and each warp runs its units through a 3-deep software pipeline:
// in iteration i it issues the row bounds and y of unit i+2, the values and
// column indices of unit i+1 (whose bounds have landed) and the x gathers of
// unit i (whose indices have landed), then sums unit i-1 (everything
// landed) while those fly.  One wait per iteration; about 3 units of loads
// in flight per warp.  Sums are per lane and per row in stored order, as in
// the other forms, so results are bitwise the reference's.  A unit with
// more than kPipeTile nonzeros is summed straight from global memory.
constexpr int kPipeTile = 256;  // nonzeros staged per unit (32 rows)

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes) {
    const unsigned s = unsigned(__cvta_generic_to_shared(smem));
    if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <class TY, class TX, class IT>
struct PipeStage {
    // row bounds and y: 4 units in flight; values, indices: 3; x: 2
    uint64_t rp[4][33];
    TY y[4][32];
    double v[3][kPipeTile];
    IT ci[3][kPipeTile];
    TX x[2][kPipeTile];
};

template <class TY, class TX, class IT, int NW>
__global__ void __launch_bounds__(NW * 32)
    csr_pipe_kernel(uint64_t rows, const uint64_t* __restrict__ rp, const IT* __restrict__ ci,
                    const double* __restrict__ v, const TX* __restrict__ x, TY* __restrict__ y) {
    extern __shared__ __align__(16) unsigned char pipe_smem[];
    using St = PipeStage<TY, TX, IT>;
    const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    St& st = reinterpret_cast<St*>(pipe_smem)[wib];
    const uint64_t units = (rows + 31) / 32;
    const uint64_t warps = uint64_t(gridDim.x) * NW;
    const uint64_t w0 = uint64_t(blockIdx.x) * NW + wib;
    const int64_t nu = w0 < units ? int64_t((units - w0 + warps - 1) / warps) : 0;
    auto unit_of = [&](int64_t i) { return w0 + uint64_t(i) * warps; };
    // the unit's nonzero range [B, E) from its staged bounds
    auto bounds = [&](int64_t i, uint64_t* B, uint64_t* E) {
        const uint64_t base = unit_of(i) * 32;
        const unsigned last = rows - base < 32 ? unsigned(rows - base) : 32u;
        *B = st.rp[i & 3][0];
        *E = st.rp[i & 3][last];
    };
    for (int64_t i = -2; i <= nu; ++i) {
        cp_async_wait_all();
        __syncwarp();
        if (i + 2 < nu) {  // row bounds and y of unit i+2
            const uint64_t base = unit_of(i + 2) * 32;
            const uint64_t r = base + lane;
            const uint64_t rr = r < rows ? r : rows;
            cp_async(&st.rp[(i + 2) & 3][lane], rp + rr, 8);
            if (lane == 0) {
                const uint64_t rl = base + 32 < rows ? base + 32 : rows;
                cp_async(&st.rp[(i + 2) & 3][32], rp + rl, 8);
            }
            if (r < rows) cp_async(&st.y[(i + 2) & 3][lane], y + r, int(sizeof(TY)));
        }
        if (i + 1 >= 0 && i + 1 < nu) {  // values and indices of unit i+1
            uint64_t B, E;
            bounds(i + 1, &B, &E);
            const unsigned cnt = unsigned(E - B);
            if (E - B <= uint64_t(kPipeTile))
                for (unsigned t = lane; t < cnt; t += 32) {
                    cp_async(&st.v[(i + 1) % 3][t], v + B + t, 8);
                    cp_async(&st.ci[(i + 1) % 3][t], ci + B + t, int(sizeof(IT)));
                }
        }
        if (i >= 0 && i < nu) {  // x gathers of unit i
            uint64_t B, E;
            bounds(i, &B, &E);
            const unsigned cnt = unsigned(E - B);
            if (E - B <= uint64_t(kPipeTile))
                for (unsigned t = lane; t < cnt; t += 32)
                    cp_async(&st.x[i & 1][t], x + st.ci[i % 3][t], int(sizeof(TX)));
        }
        cp_async_commit();
        if (i - 1 >= 0 && i - 1 < nu) {  // sum unit i-1, every operand landed
            const int64_t u = i - 1;
            const uint64_t base = unit_of(u) * 32;
            const uint64_t r = base + lane;
            uint64_t B, E;
            bounds(u, &B, &E);
            if (r < rows) {
                const uint64_t rb = st.rp[u & 3][lane], re = st.rp[u & 3][lane + 1];
                TY acc = 0;
                if (E - B <= uint64_t(kPipeTile)) {
                    const double* vs = st.v[u % 3];
                    const TX* xs = st.x[u & 1];
                    for (unsigned k = unsigned(rb - B); k < unsigned(re - B); ++k)
                        acc = acc + static_cast<TY>(vs[k]) * static_cast<TY>(xs[k]);
                } else {  // a long unit: straight from global memory
                    for (uint64_t k = rb; k < re; ++k)
                        acc = acc + static_cast<TY>(v[k]) * static_cast<TY>(x[ci[k]]);
                }
                y[r] = st.y[u & 3][lane] + acc;
            }
        }
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

bool pipelined() {
    const char* m = std::getenv("FVB_CSR_MODE");
    return m && !std::strcmp(m, "pipe");
}

template <class TY, class TX, class IT, int NW>
fvb_status launch_pipe(uint64_t rows, const uint64_t* rp, const IT* ci, const double* v,
                       const TX* x, TY* y, cudaStream_t s) {
    auto kern = csr_pipe_kernel<TY, TX, IT, NW>;
    const size_t smem = NW * sizeof(PipeStage<TY, TX, IT>);
    static const int per_sm = [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, NW * 32, smem) != cudaSuccess ||
            b < 1)
            b = 1;
        return b;
    }();
    const uint64_t units = (rows + 31) / 32;
    uint64_t grid = (units + NW - 1) / NW;
    const uint64_t cap = uint64_t(device_sm_count()) * uint64_t(per_sm);
    grid = grid < cap ? grid : cap;
    kern<<<unsigned(grid ? grid : 1), NW * 32, smem, s>>>(rows, rp, ci, v, x, y);
    return FVB_OK;
}

template <class TY, class TX, class IT>
fvb_status launch_csr(uint64_t rows, const uint64_t* rp, const IT* ci, const double* v,
                      const void* x, void* y, cudaStream_t s) {
    if (rowwise()) {
        csr_row_kernel<TY, TX, IT><<<simple_grid(rows), kCsrThreads, 0, s>>>(
            rows, rp, ci, v, static_cast<const TX*>(x), static_cast<TY*>(y));
    } else if (pipelined()) {
        const char* w = std::getenv("FVB_CSR_PIPE_WARPS");  // sweep knob: 1, 2 (default), 4
        if (w && !std::strcmp(w, "1"))
            launch_pipe<TY, TX, IT, 1>(rows, rp, ci, v, static_cast<const TX*>(x), static_cast<TY*>(y), s);
        else if (w && !std::strcmp(w, "4"))
            launch_pipe<TY, TX, IT, 4>(rows, rp, ci, v, static_cast<const TX*>(x), static_cast<TY*>(y), s);
        else
            launch_pipe<TY, TX, IT, 2>(rows, rp, ci, v, static_cast<const TX*>(x), static_cast<TY*>(y), s);
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
    // misaligned loads or stores would be a sticky device fault, not an error code
    auto misaligned = [](const void* p, size_t w) { return reinterpret_cast<uintptr_t>(p) % w != 0; };
    if (misaligned(row_ptr, 8) || misaligned(y, prec_y ? 8 : 4) ||
        (nnz && (misaligned(col_idx, sizeof(IT)) || misaligned(values, 8) ||
                 misaligned(x, prec_x ? 8 : 4))))
        return fail(FVB_EALIGN, "CSR array or plane is not element-aligned");
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
