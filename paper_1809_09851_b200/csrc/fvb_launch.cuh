// fvb_launch.cuh -- host-side launch of the fused pointwise kernel.
//
// Grid policy (measured): a one-shot tile grid -- CTA b owns
// U*256 consecutive vector groups and the grid covers the range once -- with
// 256 threads and two resident CTAs per SM where the op fits 128 registers.
// It streams HBM ~14% faster than a persistent SMs x resident-CTAs
// grid-stride sweep, which remains selectable (FVB_MODE=1) for sweeps.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <exception>
#include <new>
#include <string>

#include "fvb.h"
#include "fvb_stream.cuh"

namespace fvb {

// Per-thread error message behind fvb_last_error().
fvb_status fail(fvb_status s, const std::string& msg);
fvb_status cuda_fail(cudaError_t e, const char* what);

int device_sm_count();

// Programmatic dependent launch of the pointwise kernels (FVB_PDL=0: off).
inline bool pdl_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("FVB_PDL");
        return !(e && e[0] == '0' && e[1] == '\0');
    }();
    return v;
}

// No C++ exception crosses the C ABI: entry points whose host side
// allocates (keys, NVRTC, host threads) run their body under this guard.
template <class F>
fvb_status guarded(F&& body) noexcept {
    try {
        return body();
    } catch (const std::bad_alloc&) {
        return fail(FVB_EHOST, "host memory exhausted");
    } catch (const std::exception& e) {
        return fail(FVB_EHOST, e.what());
    } catch (...) {
        return fail(FVB_EHOST, "unexpected host-side exception");
    }
}

// Launch tuning, read once from the environment (bench sweeps only; the
// defaults are the measured best):
//   FVB_VEC      elements per access: 32 bytes (default) or half of that
//   FVB_UNROLL   groups per thread: 1 (default), 2 or 4
//   FVB_THREADS  threads per CTA: 128, 256 (default) or 512
//   FVB_MINB     __launch_bounds__ min blocks per SM: 1 (default), 2 or 4
//   FVB_MODE     1 = persistent grid-stride, 2 = one-shot tiles (default)
//   FVB_CTAS     CTAs per SM cap for the persistent mode (0 = occupancy)
// (Store policy is fixed at st.global.cs: the sweep of round 1 measured
// st.global / .cs / L1::no_allocate within 0.1% of each other.)
struct Tuning {
    int vec = 0;
    int unroll = 0;
    int threads = 0;
    int min_blocks = 0;
    int mode = 0;  // 0 = default, 1 = persistent, 2 = tiles
    int ctas_per_sm = 0;
    bool any() const { return vec || unroll || threads || min_blocks || mode; }
};
const Tuning& tuning();

template <class T>
Consts<T> make_consts(const fvb_gas* g) {
    const double gm1 = g ? g->gamma_minus_one : 2.0 / 5.0;
    const double gamma = g ? g->gamma : 7.0 / 5.0;
    const double cv = g ? g->cv : 5.0 / 2.0;
    // narrow_value: constants are rounded to the computing precision first
    // (proj/src/scalar_ops.hpp:83-85).
    return Consts<T>{static_cast<T>(0.5), static_cast<T>(gm1), static_cast<T>(gamma),
                     static_cast<T>(cv),  static_cast<T>(0.0), static_cast<T>(1.0)};
}

template <class Kernel>
int resident_ctas(Kernel k, int threads) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, 0) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    const int cap = tuning().ctas_per_sm;
    return cap > 0 && cap < per_sm ? cap : per_sm;
}

// Split [0, n) into an unaligned scalar head, V-wide groups and a scalar
// tail.  All planes must share one address residue modulo V*sizeof(T);
// returns false when they do not (caller drops to V = 1).
template <class T, int V>
bool plan_range(const void* const* ptrs, int count, uint64_t n, Range* rg) {
    const uintptr_t mod = uintptr_t(V) * sizeof(T);
    uintptr_t res = 0;
    for (int i = 0; i < count; ++i) {
        const uintptr_t r = reinterpret_cast<uintptr_t>(ptrs[i]) % mod;
        if (i == 0)
            res = r;
        else if (r != res)
            return false;
    }
    uint64_t head = res ? (mod - res) / sizeof(T) : 0;
    if (head > n) head = n;
    rg->head = head;
    rg->groups = (n - head) / V;
    rg->tail = n - head - rg->groups * V;
    return true;
}

// How the output planes of one launch overlap the planes it reads:
// kDisjoint, kSame (an output is exactly an input plane: in-place evaluation,
// as the reference allows for a destination that is also a leaf) or
// kPartial (overlapping but offset ranges: element i would read what element
// j != i writes, which no element-wise evaluation order defines).  Outputs
// that are the same plane are allowed (the later item's store wins, as in
// the reference's item order); inputs may overlap each other freely.
enum Overlap { kDisjoint = 0, kSame = 1, kPartial = 2 };

inline Overlap plane_overlap(const void* const* in, int nin, const void* const* out, int nout,
                             size_t bytes) {
    // Sort the plane starts (every plane has the same length), then compare
    // each group of identical starts with the groups that begin inside it:
    // O(P log P) for the Jacobian's 80 planes instead of all pairs.
    struct Iv {
        uintptr_t lo;
        bool out;
    };
    constexpr int kMax = 96;
    const int P = nin + nout;
    if (P > kMax) return kPartial;  // not a shape any op has
    Iv iv[kMax];
    for (int i = 0; i < nin; ++i) iv[i] = {reinterpret_cast<uintptr_t>(in[i]), false};
    for (int j = 0; j < nout; ++j) iv[nin + j] = {reinterpret_cast<uintptr_t>(out[j]), true};
    for (int i = 1; i < P; ++i) {  // insertion sort: P <= 80, mostly sorted already
        const Iv t = iv[i];
        int k = i - 1;
        while (k >= 0 && iv[k].lo > t.lo) {
            iv[k + 1] = iv[k];
            --k;
        }
        iv[k + 1] = t;
    }
    Overlap r = kDisjoint;
    for (int g = 0; g < P;) {
        int e = g;
        bool gin = false, gout = false;
        for (; e < P && iv[e].lo == iv[g].lo; ++e) (iv[e].out ? gout : gin) = true;
        if (gin && gout) r = kSame;
        for (int h = e; h < P && iv[h].lo < iv[g].lo + bytes; ++h)
            if (gout || iv[h].out) return kPartial;  // offset overlap involving a store
        g = e;
    }
    return r;
}

// An op whose output may be one of its input planes: inputs are read with
// coherent loads (the non-coherent path assumes memory no thread writes
// during the kernel).  Each element is still read before it is written by
// the one thread that owns it.
template <class Op>
struct InPlace : Op {
    static constexpr bool ALIASED = true;
};

template <class Op, class T, int V, int U, int SP, bool RED, int THREADS = 256, int MINB = 1,
          int MODE = kTiles>
fvb_status launch_fixed(const Planes<T, Op::NIN, Op::NOUT>& pl, const Consts<T>& k,
                        const Range& rg, typename Bits<T>::U* red, cudaStream_t stream) {
    auto kern = pointwise_kernel<Op, T, V, U, SP, RED, THREADS, MINB, MODE>;
    const uint64_t per_cta = uint64_t(THREADS) * U;
    uint64_t grid = (rg.groups + per_cta - 1) / per_cta;
    if (MODE == kPersistent) {
        static const int per_sm = resident_ctas(kern, THREADS);
        const uint64_t cap = uint64_t(device_sm_count()) * uint64_t(per_sm);
        grid = grid < cap ? grid : cap;
    }
    if (grid == 0) grid = 1;  // block 0 still handles the scalar head/tail
    if (grid > 0x7fffffffull) return fail(FVB_EARG, "range too large for one launch");
    // Programmatic dependent launch: back-to-back evaluations (a time step's
    // blocks, a CUDA graph of them) overlap one grid's launch with the
    // previous grid's tail; the kernel's griddepcontrol.wait keeps the
    // stream order of every byte.  FVB_PDL=0 launches plainly.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(unsigned(THREADS));
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t le = cudaLaunchKernelEx(&cfg, kern, pl, k, rg, red);
    const cudaError_t e = le != cudaSuccess ? le : cudaGetLastError();
    return e == cudaSuccess ? FVB_OK : cuda_fail(e, "kernel launch");
}

template <class T>
constexpr int vec32() {
    return int(32 / sizeof(T));
}

// Dispatch on the tuning knobs.  Only the headline kernels (TUNABLE) get the
// full variant set; everything else runs the default configuration.
// reset_red: zero the reduction word in stream order first (a fresh CFL
// maximum; the staged host path accumulates over chunks and resets it once
// itself) -- only after every plane has been validated, so a refused call
// enqueues nothing and leaves the caller's word alone.
template <class Op, class T, bool RED, bool TUNABLE>
fvb_status launch_op(const T* const* in, T* const* out, uint64_t n, const Consts<T>& k,
                     typename Bits<T>::U* red, cudaStream_t stream, bool reset_red = false) {
    auto reset = [&]() -> fvb_status {
        if (!RED || !reset_red) return FVB_OK;
        const cudaError_t e = cudaMemsetAsync(red, 0, sizeof(*red), stream);
        return e == cudaSuccess ? FVB_OK : cuda_fail(e, "lambda_max reset");
    };
    // n == 0 is a no-op even with NULL planes (an empty torch tensor or
    // DenseVector has no storage), as evaluate() returns early for n == 0;
    // a reduction over nothing is 0.
    if (n == 0) return reset();
    Planes<T, Op::NIN, Op::NOUT> pl;
    const void* ptrs[Op::NIN + (Op::NOUT > 0 ? Op::NOUT : 1)];
    int np = 0;
    for (int i = 0; i < Op::NIN; ++i) {
        if (!in[i]) return fail(FVB_EARG, "NULL input plane");
        if (reinterpret_cast<uintptr_t>(in[i]) % sizeof(T))
            return fail(FVB_EALIGN, "input plane is not element-aligned");
        pl.in[i] = in[i];
        ptrs[np++] = in[i];
    }
    for (int j = 0; j < Op::NOUT; ++j) {
        if (!out[j]) return fail(FVB_EARG, "NULL output plane");
        if (reinterpret_cast<uintptr_t>(out[j]) % sizeof(T))
            return fail(FVB_EALIGN, "output plane is not element-aligned");
        pl.out[j] = out[j];
        ptrs[np++] = out[j];
    }
    if (Op::NOUT == 0) pl.out[0] = nullptr;
    switch (plane_overlap(ptrs, Op::NIN, ptrs + Op::NIN, Op::NOUT, size_t(n) * sizeof(T))) {
        case kPartial:
            return fail(FVB_EARG, "output plane partially overlaps another plane");
        case kSame:
            if (!Op::ALIASED)
                return fail(FVB_EARG,
                            "output plane is an input plane: in-place evaluation goes through "
                            "fvb_lookup kernels");
            break;
        default:
            break;
    }
    if (fvb_status st = reset()) return st;

    constexpr int VD = vec32<T>();
    const Tuning& t = tuning();
    Range rg;
    if constexpr (TUNABLE) {
      if (t.any()) {
        // Sweep variants for the headline kernels (FVB_* environment; the
        // unset defaults below are the measured best).
        const int v = t.vec ? t.vec : VD;
        const int u = t.unroll ? t.unroll : 1;
        const int thr = t.threads ? t.threads : 256;
        const int mb = t.min_blocks ? t.min_blocks : 1;
        const int mode = t.mode ? t.mode - 1 : kTiles;
#define FVB_TRY(VV, UU, TT, MB, MD)                                                    \
    if (v == VV && u == UU && thr == TT && mb == MB && mode == MD &&                   \
        plan_range<T, VV>(ptrs, np, n, &rg))                                           \
        return launch_fixed<Op, T, VV, UU, kStoreStreaming, RED, TT, MB, MD>(pl, k, rg, red, \
                                                                             stream);
        FVB_TRY(VD, 1, 256, 1, kTiles)
        FVB_TRY(VD, 1, 256, 2, kTiles)
        FVB_TRY(VD, 2, 256, 2, kTiles)
        FVB_TRY(VD, 2, 256, 1, kTiles)
        FVB_TRY(VD, 4, 256, 1, kTiles)
        FVB_TRY(VD, 1, 128, 1, kTiles)
        FVB_TRY(VD, 2, 128, 1, kTiles)
        FVB_TRY(VD, 1, 512, 1, kTiles)
        FVB_TRY(VD / 2, 2, 256, 1, kTiles)
        FVB_TRY(VD / 2, 4, 256, 1, kTiles)
        FVB_TRY(VD / 2, 1, 256, 2, kTiles)
        FVB_TRY(1, 1, 256, 2, kTiles)
        FVB_TRY(VD / 2, 1, 128, 2, kTiles)
        FVB_TRY(VD, 1, 128, 2, kTiles)
        FVB_TRY(VD, 1, 256, 4, kTiles)
        FVB_TRY(VD / 2, 1, 256, 4, kTiles)
        FVB_TRY(VD, 1, 128, 4, kTiles)
        FVB_TRY(VD, 1, 128, 8, kTiles)
        FVB_TRY(VD, 2, 128, 4, kTiles)
        FVB_TRY(VD, 1, 256, 1, kPersistent)
        FVB_TRY(VD, 2, 256, 1, kPersistent)
#undef FVB_TRY
      }
    }
    // Default shape (measured): one-shot tiles of 256
    // threads x 1 group; two resident CTAs per SM (a 128-register cap) keep
    // 16 warps of loads in flight, except for the 32- and 75-output Jacobians,
    // whose live state would spill under that cap.
    constexpr int MB = Op::NOUT > 24 ? 1 : 2;
    // Small ranges (fewer 32-byte groups than one 256-thread CTA per SM):
    // one element per thread in 64-thread CTAs, so even n = 1024 spreads
    // over 16 SMs instead of running on one (launch-bound regime).
    if (n < uint64_t(device_sm_count()) * 256 * VD) {
        plan_range<T, 1>(ptrs, np, n, &rg);
        return launch_fixed<Op, T, 1, 1, kStoreStreaming, RED, 64, MB>(pl, k, rg, red, stream);
    }
    if (plan_range<T, VD>(ptrs, np, n, &rg)) {
        // Read-only reductions (the standalone CFL pass, 5R:0W) hide their
        // division/sqrt chains better with more, smaller CTAs: 128 threads,
        // 8 resident (64 registers): f64 0.85 -> 0.97 of peak
        // (profiles/r01_cfl_sweep.txt).
        if constexpr (Op::NOUT == 0)
            return launch_fixed<Op, T, VD, 1, kStoreStreaming, RED, 128, 8>(pl, k, rg, red, stream);
        return launch_fixed<Op, T, VD, 1, kStoreStreaming, RED, 256, MB>(pl, k, rg, red, stream);
    }
    // Planes with different 32-byte residues: element-wide accesses.
    plan_range<T, 1>(ptrs, np, n, &rg);
    return launch_fixed<Op, T, 1, 1, kStoreStreaming, RED, 256, MB>(pl, k, rg, red, stream);
}

}  // namespace fvb
