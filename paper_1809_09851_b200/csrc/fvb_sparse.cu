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
// the comparison in tools/csr_bench.py via FVB_CSR_ROWWISE=1).
template <class TY, class TX>
__global__ void __launch_bounds__(kCsrThreads)
    csr_row_kernel(uint64_t rows, const uint64_t* __restrict__ rp, const uint64_t* __restrict__ ci,
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
template <class TY, class TX, int MINB, int UNR>
__global__ void __launch_bounds__(kCsrThreads, MINB)
    csr_warp_kernel(uint64_t rows, const uint64_t* __restrict__ rp,
                    const uint64_t* __restrict__ ci, const double* __restrict__ v,
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
            const uint64_t* cb = ci + base;
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

// ---- bulk-copy ring (TMA 1-D bulk copies into shared memory) ----
//
// The warp-staged form issues the value/index loads and the x gathers from
// the same threads: every round waits for HBM (the indices) and then for L2
// (the gathers) back to back, and the bytes in flight per SM are bounded by
// registers.  Here the unit of work is one warp's 32 rows, whose nonzeros
// are one contiguous range.  A producer warp streams each unit's values,
// column indices and row pointers into one of NS shared-memory stages with
// cp.async.bulk (the copy engine holds the bytes in flight, not registers),
// completing on the stage's "full" mbarrier.  NW consumer warps take units
// round-robin: wait "full", gather x for up to kCsrPer entries per lane,
// park the products over the stage's values, and each lane sums its row in
// stored order -- the same two roundings per product and the same
// left-to-right additions as csr_matvec_acc_t -- then arrive on "empty".
//
// Phase bookkeeping: mbarrier waits are by parity, so no waiter may run two
// phases ahead.  Stage s is always consumed by the same warp (NS % NW == 0),
// and the producer's lanes fill units in lock-step rounds of kCsrRound with
// NS >= kCsrRound, so every stage's pending phase is the one its waiter
// expects.  The producer loads the row bounds of 32 units at once, one group
// ahead, so the HBM latency of rp is off the issue path.
//
// Bulk copies need 16-byte aligned addresses and sizes, and the C ABI takes
// any naturally aligned plane: the element before the first 16-byte boundary
// of a range (the "head") and the one after the last (the "tail") are read
// from global memory directly, so nothing outside [rp[r0], rp[r1]) and
// rp[r0..r1] is ever touched.  A unit whose range exceeds a stage (32 *
// kCsrPer nonzeros) is summed row by row from global memory instead.

constexpr int kCsrPer = 8;    // stage entries per lane: 256 nonzeros per 32 rows
constexpr int kCsrRound = 8;  // producer lanes filling stages at once

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "FVB_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra FVB_WAIT_%=;\n}" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}
// global -> this CTA's shared memory, completion counted on mbarrier b;
// evict-first in L2 so the streamed CSR arrays do not push x out
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(b)), "l"(policy)
        : "memory");
}

// One stage's bookkeeping, written by the producer lane before its arrive
// (release) and read by the consumer warp after its wait (acquire).
struct CsrStageMeta {
    uint64_t beg, end;      // nonzero range [beg, end) = [rp[r0], rp[r1]) of the unit
    uint64_t v0, v1;        // values [v0, v1) are in the stage (slot k - v0)
    uint64_t c0, c1;        // column indices [c0, c1) likewise
    uint64_t p0, p1;        // row pointers [p0, p1) likewise
    uint32_t direct;        // 1: range exceeds the stage, rows summed from global
    uint32_t pad;
};

// [ceil16(addr(lo)), floor16(addr(hi))) as element indices of an 8-byte array
__device__ __forceinline__ void aligned_span(const void* base, uint64_t lo, uint64_t hi,
                                             uint64_t& a, uint64_t& b) {
    const uint64_t p = reinterpret_cast<uint64_t>(base);
    a = lo + (((p + 8 * lo) & 15) ? 1 : 0);
    b = hi - (((p + 8 * hi) & 15) ? 1 : 0);
    if (lo >= hi || b < a) b = a = lo;  // nothing bulk-copyable
}

template <class TY, int NW, int NS>
struct CsrRing {
    static constexpr int kCap = 32 * kCsrPer;
    double v[NS][kCap];
    uint64_t c[NS][kCap];
    uint64_t rp[NS][34];  // rp[r0 .. r0+32] (+1 for the alignment shift)
    CsrStageMeta meta[NS];
    uint64_t full[NS], empty[NS];
};

template <class TY, class TX, int NW, int NS>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    csr_bulk_kernel(uint64_t rows, const uint64_t* __restrict__ rp, const uint64_t* __restrict__ ci,
                    const double* __restrict__ v, const TX* __restrict__ x, TY* __restrict__ y) {
    static_assert(NS % NW == 0 && NS >= 2 * kCsrRound, "parity bookkeeping (see above)");
    using Ring = CsrRing<TY, NW, NS>;
    constexpr uint64_t kCap = Ring::kCap;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Ring& R = *reinterpret_cast<Ring*>(smem_raw);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t units = (rows + 31) / 32;
    const uint64_t G = gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&R.full[s], 1);
            mbar_init(&R.empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NW) {
        // ---- producer: the row bounds of 32 items per load (prefetched one
        // group ahead), issued in lock-step rounds of 8 lanes ----
        uint64_t policy;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
        auto bounds = [&](uint64_t j, uint64_t& b, uint64_t& e) {
            const uint64_t u = blockIdx.x + j * G;
            b = e = 0;
            if (u < units) {
                const uint64_t r0 = u * 32, r1 = r0 + 32 < rows ? r0 + 32 : rows;
                b = rp[r0];
                e = rp[r1];
            }
        };
        uint64_t nb, ne;
        bounds(lane, nb, ne);
        for (uint64_t j0 = 0; blockIdx.x + j0 * G < units; j0 += 32) {
            const uint64_t gb = nb, ge = ne;
            bounds(j0 + 32 + lane, nb, ne);  // next group, in flight meanwhile
            for (unsigned q = 0; q < 32; q += kCsrRound) {
                const unsigned src = q + (lane % kCsrRound);
                const uint64_t b = __shfl_sync(0xffffffffu, gb, src);
                const uint64_t e = __shfl_sync(0xffffffffu, ge, src);
                const uint64_t j = j0 + src;
                const uint64_t u = blockIdx.x + j * G;
                if (lane < kCsrRound && u < units) {
                    const int s = int(j % NS);
                    if (j >= uint64_t(NS)) mbar_wait(&R.empty[s], uint32_t((j / NS - 1) & 1));
                    const uint64_t r0 = u * 32, r1 = r0 + 32 < rows ? r0 + 32 : rows;
                    CsrStageMeta& m = R.meta[s];
                    m.beg = b;
                    m.end = e;
                    m.direct = e - b > kCap;
                    aligned_span(rp, r0, r1 + 1, m.p0, m.p1);
                    uint32_t bytes = uint32_t(8 * (m.p1 - m.p0));
                    if (!m.direct) {
                        aligned_span(v, b, e, m.v0, m.v1);
                        aligned_span(ci, b, e, m.c0, m.c1);
                        bytes += uint32_t(8 * ((m.v1 - m.v0) + (m.c1 - m.c0)));
                    } else {
                        m.v0 = m.v1 = m.c0 = m.c1 = b;
                    }
                    if (bytes) {
                        mbar_arrive_tx(&R.full[s], bytes);
                        if (m.v1 > m.v0)
                            bulk_g2s(R.v[s], v + m.v0, uint32_t(8 * (m.v1 - m.v0)), &R.full[s],
                                     policy);
                        if (m.c1 > m.c0)
                            bulk_g2s(R.c[s], ci + m.c0, uint32_t(8 * (m.c1 - m.c0)), &R.full[s],
                                     policy);
                        if (m.p1 > m.p0)
                            bulk_g2s(R.rp[s], rp + m.p0, uint32_t(8 * (m.p1 - m.p0)), &R.full[s],
                                     policy);
                    } else {
                        mbar_arrive(&R.full[s]);
                    }
                }
                __syncwarp();  // lock-step rounds (phase bookkeeping)
            }
        }
        return;
    }

    // ---- consumer warp `warp`: items j = warp, warp + NW, ... ----
    for (uint64_t j = warp; blockIdx.x + j * G < units; j += NW) {
        const uint64_t u = blockIdx.x + j * G;
        const int s = int(j % NS);
        const uint64_t r0 = u * 32, r1 = r0 + 32 < rows ? r0 + 32 : rows;
        const uint64_t r = r0 + lane;
        const bool valid = r < rows;
        const TY yv = valid ? y[r] : TY(0);  // independent of the stage: before the wait
        mbar_wait(&R.full[s], uint32_t((j / NS) & 1));
        const CsrStageMeta& m = R.meta[s];
        const uint64_t* rps = R.rp[s];
        auto rp_at = [&](uint64_t i) {  // the unit's first/last pointers are beg/end
            return i == r0 ? m.beg : (i == r1 ? m.end : rps[i - m.p0]);
        };
        const uint64_t rb = valid ? rp_at(r) : 0, re = valid ? rp_at(r + 1) : 0;
        TY acc = 0;
        if (!m.direct) {
            const double* vs = R.v[s];
            const uint64_t* cs = R.c[s];
            const unsigned lim = unsigned(m.end - m.beg);  // <= kCap
            TX xv[kCsrPer];
#pragma unroll
            for (int t = 0; t < kCsrPer; ++t) {
                const unsigned q = lane + 32u * t;
                const uint64_t k = m.beg + q;
                if (q < lim) xv[t] = x[(k >= m.c0 && k < m.c1) ? cs[k - m.c0] : ci[k]];
            }
            double val[kCsrPer];
#pragma unroll
            for (int t = 0; t < kCsrPer; ++t) {
                const unsigned q = lane + 32u * t;
                const uint64_t k = m.beg + q;
                if (q < lim) val[t] = (k >= m.v0 && k < m.v1) ? vs[k - m.v0] : v[k];
            }
            // every value read: the products overwrite the value slots
            // (product q = entry beg + q at slot q)
            __syncwarp();
            TY* p = reinterpret_cast<TY*>(R.v[s]);
#pragma unroll
            for (int t = 0; t < kCsrPer; ++t)
                if (lane + 32u * t < lim)
                    p[lane + 32u * t] = static_cast<TY>(val[t]) * static_cast<TY>(xv[t]);
            __syncwarp();
            for (uint64_t k = rb; k < re; ++k) acc = acc + p[k - m.beg];
        } else {
            for (uint64_t k = rb; k < re; ++k)
                acc = acc + static_cast<TY>(v[k]) * static_cast<TY>(x[ci[k]]);
        }
        if (valid) y[r] = yv + acc;
        // the products were written through the generic proxy into memory
        // the copy engine refills next: order them before the release
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&R.empty[s]);
    }
}

enum class CsrMode { kAuto, kRow, kWarp, kBulk };

// FVB_CSR_MODE = row | warp | bulk forces a form (tools/csr_bench.py);
// FVB_CSR_ROWWISE=1 is the older spelling of row.  Read per call so tests
// can cover every form in one process.
CsrMode csr_mode() {
    const char* e = std::getenv("FVB_CSR_MODE");
    if (e && *e) {
        if (!std::strcmp(e, "row")) return CsrMode::kRow;
        if (!std::strcmp(e, "warp")) return CsrMode::kWarp;
        if (!std::strcmp(e, "bulk")) return CsrMode::kBulk;
    }
    const char* r = std::getenv("FVB_CSR_ROWWISE");
    if (r && *r && *r != '0') return CsrMode::kRow;
    return CsrMode::kAuto;
}

// Default ring shape (consumer warps, stages); others are instantiated for
// f64 only, for tools/csr_bench.py sweeps (FVB_CSR_BULK=<NW>x<NS>).
constexpr int kBulkNW = 16, kBulkNS = 32;

template <class TY, class TX, int NW, int NS>
fvb_status launch_csr_bulk_shape(uint64_t rows, const uint64_t* rp, const uint64_t* ci,
                                 const double* v, const TX* x, TY* y, cudaStream_t st) {
    auto k = csr_bulk_kernel<TY, TX, NW, NS>;
    constexpr size_t smem = sizeof(CsrRing<TY, NW, NS>);
    static thread_local int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {
        const cudaError_t e =
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return cuda_fail(e, "csr bulk smem attribute");
        configured = dev;
    }
    const uint64_t units = (rows + 31) / 32;
    const uint64_t cap = uint64_t(device_sm_count());  // one resident CTA per SM
    const unsigned g = unsigned(units < cap ? units : cap);
    k<<<g, 32 * (NW + 1), smem, st>>>(rows, rp, ci, v, x, y);
    return FVB_OK;
}

template <class TY, class TX>
fvb_status launch_csr_bulk(uint64_t rows, const uint64_t* rp, const uint64_t* ci, const double* v,
                           const TX* x, TY* y, cudaStream_t s) {
    if constexpr (sizeof(TY) == 8 && sizeof(TX) == 8) {
        const char* e = std::getenv("FVB_CSR_BULK");
        if (e && *e) {
            if (!std::strcmp(e, "16x48"))
                return launch_csr_bulk_shape<TY, TX, 16, 48>(rows, rp, ci, v, x, y, s);
            if (!std::strcmp(e, "24x48"))
                return launch_csr_bulk_shape<TY, TX, 24, 48>(rows, rp, ci, v, x, y, s);
            if (!std::strcmp(e, "20x40"))
                return launch_csr_bulk_shape<TY, TX, 20, 40>(rows, rp, ci, v, x, y, s);
            if (!std::strcmp(e, "8x32"))
                return launch_csr_bulk_shape<TY, TX, 8, 32>(rows, rp, ci, v, x, y, s);
        }
    }
    return launch_csr_bulk_shape<TY, TX, kBulkNW, kBulkNS>(rows, rp, ci, v, x, y, s);
}

template <class TY, class TX>
fvb_status launch_csr(uint64_t rows, uint64_t nnz, const uint64_t* rp, const uint64_t* ci,
                      const double* v, const void* x, void* y, cudaStream_t s) {
    CsrMode mode = csr_mode();
    if (mode == CsrMode::kAuto) {
        // the bulk pipeline when a row block's range usually fits one stage
        // (stencil-like rows) and the arrays are naturally aligned
        const bool aligned = !(reinterpret_cast<uintptr_t>(ci) & 7) &&
                             !(reinterpret_cast<uintptr_t>(v) & 7);
        mode = aligned && nnz <= rows * uint64_t(kCsrPer * 7 / 8) ? CsrMode::kBulk
                                                                   : CsrMode::kWarp;
    }
    if (mode == CsrMode::kBulk) {
        const fvb_status st = launch_csr_bulk<TY, TX>(rows, rp, ci, v, static_cast<const TX*>(x),
                                                      static_cast<TY*>(y), s);
        if (st != FVB_OK) return st;
    } else if (mode == CsrMode::kRow) {
        csr_row_kernel<TY, TX><<<simple_grid(rows), kCsrThreads, 0, s>>>(
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
        // 8 resident CTAs (32 registers) and two tile entries in flight per
        // lane: the measured best (profiles/r01_csr_shapes.txt)
        csr_warp_kernel<TY, TX, 8, 2><<<g, kCsrThreads, 0, s>>>(rows, rp, ci, v, xx, yy);
    }
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
        return prec_x == FVB_F64 ? launch_csr<double, double>(rows, nnz, row_ptr, col_idx, values, x, y, s)
                                 : launch_csr<double, float>(rows, nnz, row_ptr, col_idx, values, x, y, s);
    return prec_x == FVB_F64 ? launch_csr<float, double>(rows, nnz, row_ptr, col_idx, values, x, y, s)
                             : launch_csr<float, float>(rows, nnz, row_ptr, col_idx, values, x, y, s);
}

}  // extern "C"
