// fvb_host.cu -- the host-buffer (end-to-end) path: fvb_ctx and the
// streamed fvb_flux_host / fvb_jacobian_host.
//
// The reference evaluates host DenseVectors in place (proj/src/
// backend_eval.cpp:280-346).  A drop-in device backend handed host buffers
// must move them over PCIe; this path hides the kernel entirely behind the
// copies: the range is cut into chunks, and chunk c runs on slot c % kSlots
// as [H2D inputs -> fused kernel -> D2H outputs] in that slot's stream, so
// the H2D of one chunk, the kernel of another and the D2H of a third overlap
// on the two copy directions.  Slot buffers are reused in stream order; the
// host synchronises once, at the end.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "fvb.h"
#include "fvb_launch.cuh"

struct fvb_ctx {
    static constexpr int kSlots = 3;
    int device = 0;
    uint64_t chunk_points = 0;  // 0 = size chunks by bytes
    cudaStream_t stream[kSlots] = {};
    void* slot_buf[kSlots] = {};
    size_t slot_bytes = 0;
    void* red = nullptr;  // lambda-max accumulator (8 bytes)
    cudaEvent_t reset_done = nullptr;
};

namespace fvb {
namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

fvb_status ensure_slots(fvb_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->slot_bytes) return FVB_OK;
    for (int s = 0; s < fvb_ctx::kSlots; ++s) {
        if (ctx->slot_buf[s]) {
            cudaStreamSynchronize(ctx->stream[s]);
            cudaFree(ctx->slot_buf[s]);
            ctx->slot_buf[s] = nullptr;
        }
    }
    ctx->slot_bytes = 0;
    for (int s = 0; s < fvb_ctx::kSlots; ++s) {
        const cudaError_t e = cudaMalloc(&ctx->slot_buf[s], bytes);
        if (e != cudaSuccess) return cuda_fail(e, "staging allocation");
    }
    ctx->slot_bytes = bytes;
    return FVB_OK;
}

// Chunk size: 256 MiB of planes per slot unless the context fixes it.
uint64_t chunk_for(const fvb_ctx* ctx, size_t bytes_per_point, uint64_t n) {
    uint64_t c = ctx->chunk_points;
    if (!c) c = (uint64_t(256) << 20) / bytes_per_point;
    c = std::max<uint64_t>(c & ~uint64_t(255), 256);  // keep 32-byte alignment of slot planes
    return std::min<uint64_t>(c, std::max<uint64_t>(n, 1));
}

// Host threads copying pass-through items: output j < PASS is bit-for-bit
// input plane 1 + j (the flux's row 0 is the momentum fields themselves,
// include/fusevec/fluid.hpp:168-169).  The host already holds those bytes,
// so they are copied host-side, concurrently with the device pipeline,
// instead of crossing PCIe twice.  Joined on every exit path.
struct PassThrough {
    std::vector<std::thread> workers;
    PassThrough(const void* const* in, void* const* out, int pass, size_t bytes) {
        if (pass <= 0 || bytes == 0) return;
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned nt = std::min(8u, std::max(1u, hw / 2));
        const size_t total = size_t(pass) * bytes;
        const size_t per = (total + nt - 1) / nt;
        auto copy = [=](size_t lo, size_t hi) {
            while (lo < hi) {
                const size_t plane = lo / bytes, at = lo % bytes;
                const size_t len = std::min(hi - lo, bytes - at);
                std::memcpy(static_cast<char*>(out[plane]) + at,
                            static_cast<const char*>(in[1 + plane]) + at, len);
                lo += len;
            }
        };
        try {
            for (unsigned t = 0; t < nt; ++t) {
                const size_t lo = size_t(t) * per;
                workers.emplace_back(copy, lo, std::min(total, lo + per));
            }
        } catch (...) {  // no threads to be had: copy on the calling thread
            for (auto& w : workers) w.join();
            workers.clear();
            copy(0, total);
        }
    }
    ~PassThrough() {
        for (auto& w : workers) w.join();
    }
};

template <class Op, class T, bool RED, bool TUNE, int PASS = 0>
fvb_status pipeline(fvb_ctx* ctx, const void* const* in, void* const* out, uint64_t n,
                    const Consts<T>& k, double* lambda_max) {
    constexpr int NIN = Op::NIN, NOUT = Op::NOUT;
    if (!in || !out) return fail(FVB_EARG, "NULL plane array");
    for (int i = 0; i < NIN; ++i)
        if (!in[i]) return fail(FVB_EARG, "NULL input plane");
    for (int j = 0; j < NOUT; ++j)
        if (!out[j]) return fail(FVB_EARG, "NULL output plane");
    // The chunks of different slots read and write concurrently, and the
    // pass-through threads copy host-side: host outputs must be disjoint
    // from the inputs.
    if (plane_overlap(in, NIN, const_cast<const void* const*>(out), NOUT, size_t(n) * sizeof(T)) !=
        kDisjoint)
        return fail(FVB_EARG, "host output plane overlaps an input plane");
    DeviceGuard guard(ctx->device);
    using Bu = typename Bits<T>::U;
    if (RED) {
        cudaError_t e = cudaMemsetAsync(ctx->red, 0, sizeof(Bu), ctx->stream[0]);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->reset_done, ctx->stream[0]);
        for (int s = 1; s < fvb_ctx::kSlots && e == cudaSuccess; ++s)
            e = cudaStreamWaitEvent(ctx->stream[s], ctx->reset_done, 0);
        if (e != cudaSuccess) return cuda_fail(e, "lambda reset");
    }
    if (n == 0) {
        if (RED && lambda_max) *lambda_max = 0.0;
        return FVB_OK;
    }
    const uint64_t chunk = chunk_for(ctx, sizeof(T) * (NIN + NOUT), n);
    if (fvb_status st = ensure_slots(ctx, size_t(chunk) * sizeof(T) * (NIN + NOUT))) return st;

    PassThrough pass(in, out, PASS, size_t(n) * sizeof(T));
    const uint64_t nchunks = (n + chunk - 1) / chunk;
    for (uint64_t c = 0; c < nchunks; ++c) {
        const int slot = int(c % fvb_ctx::kSlots);
        cudaStream_t s = ctx->stream[slot];
        const uint64_t off = c * chunk;
        const uint64_t cnt = std::min(chunk, n - off);
        const size_t bytes = size_t(cnt) * sizeof(T);
        T* base = static_cast<T*>(ctx->slot_buf[slot]);
        const T* din[NIN];
        T* dout[NOUT > 0 ? NOUT : 1];
        for (int i = 0; i < NIN; ++i) {
            T* d = base + size_t(i) * chunk;
            din[i] = d;
            const cudaError_t e = cudaMemcpyAsync(d, static_cast<const T*>(in[i]) + off, bytes,
                                                  cudaMemcpyHostToDevice, s);
            if (e != cudaSuccess) return cuda_fail(e, "host->device copy");
        }
        for (int j = 0; j < NOUT; ++j) dout[j] = base + size_t(NIN + j) * chunk;
        fvb_status st = launch_op<Op, T, RED, TUNE>(din, dout, cnt, k,
                                                    static_cast<Bu*>(ctx->red), s);
        if (st) return st;
        for (int j = PASS; j < NOUT; ++j) {
            const cudaError_t e = cudaMemcpyAsync(static_cast<T*>(out[j]) + off, dout[j], bytes,
                                                  cudaMemcpyDeviceToHost, s);
            if (e != cudaSuccess) return cuda_fail(e, "device->host copy");
        }
    }
    for (int s = 0; s < fvb_ctx::kSlots; ++s) {
        const cudaError_t e = cudaStreamSynchronize(ctx->stream[s]);
        if (e != cudaSuccess) return cuda_fail(e, "pipeline completion");
    }
    if (RED && lambda_max) {
        Bu bits = 0;
        const cudaError_t e = cudaMemcpy(&bits, ctx->red, sizeof(Bu), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(e, "lambda_max read-back");
        T v;
        std::memcpy(&v, &bits, sizeof v);
        *lambda_max = double(v);
    }
    return FVB_OK;
}

// PASS_DIM: the first d outputs are pass-through copies of inputs 1..d.
template <template <class, int> class OpT, bool RED, class T, bool TUNE3 = false,
          bool PASS_DIM = false>
fvb_status pipeline_dim(fvb_ctx* ctx, const fvb_gas* gas, uint32_t dim, const void* const* in,
                        void* const* out, uint64_t n, double* lambda_max) {
    const auto k = make_consts<T>(gas);
    switch (dim) {
        case 1:
            return pipeline<OpT<T, 1>, T, RED, false, PASS_DIM ? 1 : 0>(ctx, in, out, n, k,
                                                                        lambda_max);
        case 2:
            return pipeline<OpT<T, 2>, T, RED, false, PASS_DIM ? 2 : 0>(ctx, in, out, n, k,
                                                                        lambda_max);
        default:
            return pipeline<OpT<T, 3>, T, RED, TUNE3, PASS_DIM ? 3 : 0>(ctx, in, out, n, k,
                                                                        lambda_max);
    }
}

fvb_status check(fvb_ctx* ctx, const fvb_gas* gas, uint32_t dim, uint8_t prec) {
    if (!ctx) return fail(FVB_EARG, "NULL context");
    if (prec > 1) return fail(FVB_EPREC, "precision code must be 0 (f32) or 1 (f64)");
    if (dim < 1 || dim > 3) return fail(FVB_EARG, "dim must be 1, 2 or 3");
    if (gas && (!(gas->cv > 0) || !(gas->gamma_minus_one > 0) || !(gas->gamma > 1)))
        return fail(FVB_EARG, "gas constants must satisfy cv > 0, gamma-1 > 0, gamma > 1");
    return FVB_OK;
}

}  // namespace
}  // namespace fvb

using namespace fvb;

extern "C" {

fvb_status fvb_ctx_create(int device, uint64_t chunk_points, fvb_ctx** out) {
    if (!out) return fail(FVB_EARG, "NULL output");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, "device query");
    if (device < 0 || device >= count) return fail(FVB_EARG, "device ordinal out of range");
    auto* ctx = new (std::nothrow) fvb_ctx;
    if (!ctx) return fail(FVB_EHOST, "out of host memory");
    ctx->device = device;
    ctx->chunk_points = chunk_points;
    DeviceGuard guard(device);
    for (int s = 0; s < fvb_ctx::kSlots && e == cudaSuccess; ++s)
        e = cudaStreamCreateWithFlags(&ctx->stream[s], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->red, 8);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->reset_done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        fvb_ctx_destroy(ctx);
        return cuda_fail(e, "context creation");
    }
    *out = ctx;
    return FVB_OK;
}

fvb_status fvb_ctx_destroy(fvb_ctx* ctx) {
    if (!ctx) return FVB_OK;
    DeviceGuard guard(ctx->device);
    for (int s = 0; s < fvb_ctx::kSlots; ++s) {
        if (ctx->stream[s]) cudaStreamSynchronize(ctx->stream[s]);
        if (ctx->slot_buf[s]) cudaFree(ctx->slot_buf[s]);
        if (ctx->stream[s]) cudaStreamDestroy(ctx->stream[s]);
    }
    if (ctx->red) cudaFree(ctx->red);
    if (ctx->reset_done) cudaEventDestroy(ctx->reset_done);
    delete ctx;
    return FVB_OK;
}

fvb_status fvb_flux_host(fvb_ctx* ctx, const fvb_gas* gas, uint32_t dim, uint8_t prec,
                         uint64_t n, const void* const* in, void* const* out) {
    return guarded([&]() -> fvb_status {
        if (fvb_status st = check(ctx, gas, dim, prec)) return st;
        if (prec == FVB_F64)
            return pipeline_dim<FluxOp, false, double, true, true>(ctx, gas, dim, in, out, n, nullptr);
        return pipeline_dim<FluxOp, false, float, true, true>(ctx, gas, dim, in, out, n, nullptr);
    });
}

fvb_status fvb_jacobian_host(fvb_ctx* ctx, const fvb_gas* gas, uint32_t dim, uint8_t prec,
                             uint64_t n, const void* const* in, void* const* out,
                             double* lambda_max) {
    return guarded([&]() -> fvb_status {
        if (fvb_status st = check(ctx, gas, dim, prec)) return st;
        if (prec == FVB_F64) {
            if (lambda_max)
                return pipeline_dim<JacobianOp, true, double>(ctx, gas, dim, in, out, n, lambda_max);
            return pipeline_dim<JacobianOp, false, double>(ctx, gas, dim, in, out, n, nullptr);
        }
        if (lambda_max)
            return pipeline_dim<JacobianOp, true, float>(ctx, gas, dim, in, out, n, lambda_max);
        return pipeline_dim<JacobianOp, false, float>(ctx, gas, dim, in, out, n, nullptr);
    });
}

}  // extern "C"
