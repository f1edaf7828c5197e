// fvb_host.cu -- the host-buffer (end-to-end) path: fvb_ctx, the staged
// executor behind it, and fvb_flux_host / fvb_jacobian_host /
// fvb_launch_host.
//
// The reference evaluates host DenseVectors in place (proj/src/
// backend_eval.cpp:280-346).  A drop-in device backend handed host buffers
// must move them over PCIe; this path hides the kernel behind the copies.
// The range is cut into chunks, and chunk c runs on slot c % slots as
// [H2D inputs -> fused kernel -> D2H outputs] in that slot's stream, so the
// H2D of one chunk, the kernel of another and the D2H of a third overlap on
// the two copy directions.
//
// Host planes may be pinned or pageable (the reference's DenseVectors are
// ordinary heap memory).  Pinned planes are DMA'd directly.  Pageable ones
// go through pinned bounce buffers of the slot: a pool of host threads packs
// chunk c's pageable inputs while the device still works on chunks c-1 and
// c-2, and unpacks a chunk's outputs once its D2H has completed.  Device
// planes (resident leaves, device destinations) are used in place.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "fvb.h"
#include "fvb_hostcopy.h"
#include "fvb_launch.cuh"

namespace fvb {
namespace {

// ---- a small pool of copy threads -------------------------------------------------

struct Piece {
    char* dst;
    const char* src;
    size_t bytes;
};

class CopyPool {
  public:
    explicit CopyPool(unsigned workers) {
        try {
            for (unsigned t = 0; t < workers; ++t) threads_.emplace_back([this] { loop(); });
        } catch (...) {  // fewer threads than asked: the caller still copies
            stop_workers();
        }
    }
    ~CopyPool() { stop_workers(); }

    // Every piece copied when this returns; the calling thread helps.
    void run(const std::vector<Piece>& pieces) {
        if (pieces.empty()) return;
        size_t total = 0;
        for (const Piece& p : pieces) total += p.bytes;
        // waking the workers costs more than copying a few hundred KiB
        if (threads_.empty() || pieces.size() == 1 || total < (size_t(1) << 20)) {
            for (const Piece& p : pieces) host_copy(p.dst, p.src, p.bytes);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            work_ = &pieces;
            next_.store(0);
            pending_ = unsigned(threads_.size());
            ++gen_;
        }
        cv_.notify_all();
        drain(pieces);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
        work_ = nullptr;
    }

  private:
    void drain(const std::vector<Piece>& pieces) {
        for (size_t i; (i = next_.fetch_add(1)) < pieces.size();)
            host_copy(pieces[i].dst, pieces[i].src, pieces[i].bytes);
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            const std::vector<Piece>* w = work_;
            lk.unlock();
            drain(*w);
            lk.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }
    void stop_workers() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
        threads_.clear();
    }

    std::mutex mu_;
    std::condition_variable cv_, done_;
    std::vector<std::thread> threads_;
    const std::vector<Piece>* work_ = nullptr;
    std::atomic<size_t> next_{0};
    unsigned pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

}  // namespace
}  // namespace fvb

struct fvb_ctx {
    static constexpr int kMaxSlots = 8;
    int slots = 3;  // pipeline depth (FVB_HOST_SLOTS, 2..8; a sweep knob)
    int device = 0;
    uint64_t chunk_points = 0;  // 0 = size chunks by bytes
    cudaStream_t stream[kMaxSlots] = {};
    cudaEvent_t done[kMaxSlots] = {};  // the slot's last D2H has completed
    void* slot_buf[kMaxSlots] = {};    // device staging
    size_t slot_bytes = 0;
    void* pin_buf[kMaxSlots] = {};     // pinned bounce buffers for pageable planes
    size_t pin_bytes = 0;
    void* red = nullptr;            // lambda-max accumulator (8 bytes)
    cudaEvent_t reset_done = nullptr;
    std::unique_ptr<fvb::CopyPool> pool;
};

namespace fvb {
namespace {

// Sweep knobs of the host side (tools/gpu_e2e_jac_sweep.sh; unset = the
// measured defaults): FVB_FILL_THREADS (host-side fills and pass-through
// copies), FVB_POOL_THREADS (bounce and duplicate copies), FVB_DUPS_ON_LINK=1
// (the Jacobian's duplicate entries shipped over PCIe instead of copied).
int env_knob(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

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

// Device staging (required) and pinned bounce buffers (optional: *pinned is
// false when the host has no pinned memory to give; the caller then copies
// pageable planes with plain cudaMemcpyAsync, slower but correct).
fvb_status ensure_buffers(fvb_ctx* ctx, size_t dev_bytes, size_t pin_bytes, bool* pinned) {
    *pinned = true;
    if (dev_bytes > ctx->slot_bytes || pin_bytes > ctx->pin_bytes) {
        for (int s = 0; s < ctx->slots; ++s) cudaStreamSynchronize(ctx->stream[s]);
    }
    if (dev_bytes > ctx->slot_bytes) {
        for (int s = 0; s < ctx->slots; ++s) {
            if (ctx->slot_buf[s]) cudaFree(ctx->slot_buf[s]);
            ctx->slot_buf[s] = nullptr;
        }
        ctx->slot_bytes = 0;
        for (int s = 0; s < ctx->slots; ++s) {
            const cudaError_t e = cudaMalloc(&ctx->slot_buf[s], dev_bytes);
            if (e != cudaSuccess) return cuda_fail(e, "staging allocation");
        }
        ctx->slot_bytes = dev_bytes;
    }
    if (pin_bytes > ctx->pin_bytes) {
        for (int s = 0; s < ctx->slots; ++s) {
            if (ctx->pin_buf[s]) cudaFreeHost(ctx->pin_buf[s]);
            ctx->pin_buf[s] = nullptr;
        }
        ctx->pin_bytes = 0;
        for (int s = 0; s < ctx->slots; ++s) {
            if (cudaHostAlloc(&ctx->pin_buf[s], pin_bytes, cudaHostAllocDefault) != cudaSuccess) {
                cudaGetLastError();  // not sticky: fall back to unbounced copies
                for (int q = 0; q <= s; ++q) {
                    if (ctx->pin_buf[q]) cudaFreeHost(ctx->pin_buf[q]);
                    ctx->pin_buf[q] = nullptr;
                }
                *pinned = false;
                return FVB_OK;
            }
        }
        ctx->pin_bytes = pin_bytes;
    }
    return FVB_OK;
}

// Chunk size: 256 MiB of device staging per slot unless the context fixes it.
uint64_t chunk_for(const fvb_ctx* ctx, size_t bytes_per_point, uint64_t n) {
    uint64_t c = ctx->chunk_points;
    if (!c) c = (uint64_t(256) << 20) / std::max<size_t>(bytes_per_point, 1);
    c = std::max<uint64_t>(c & ~uint64_t(255), 256);  // keep 32-byte alignment of slot planes
    // a range shorter than one chunk still strides its slot planes by a
    // multiple of 256 elements, so every plane keeps the 32-byte residue
    return std::min<uint64_t>(c, (std::max<uint64_t>(n, 1) + 255) & ~uint64_t(255));
}

enum class Mem { kPageable, kPinned, kDevice };

Mem memory_kind(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // clear: unknown memory is pageable
        return Mem::kPageable;
    }
    switch (a.type) {
        case cudaMemoryTypeHost:
        case cudaMemoryTypeManaged: return Mem::kPinned;
        case cudaMemoryTypeDevice: return Mem::kDevice;
        default: return Mem::kPageable;
    }
}

// Host threads write (and read) host planes before staged() classifies
// them, so a device pointer handed over as a host plane is refused first:
// on the host it would be a wild access, not an error code.
fvb_status host_planes(const void* const* p, size_t count, size_t width) {
    for (size_t i = 0; i < count; ++i) {
        if (p[i] && reinterpret_cast<uintptr_t>(p[i]) % width)
            return fail(FVB_EALIGN, "host plane is not element-aligned");
        if (p[i] && memory_kind(p[i]) == Mem::kDevice)
            return fail(FVB_EARG, "a host plane is device memory");
    }
    return FVB_OK;
}

// One plane of a staged launch.
struct Arg {
    char* host = nullptr;  // host plane (pinned or pageable), or
    char* dev = nullptr;   // a device plane used in place; both NULL = NULL slot
    size_t width = 8;
    bool out = false;
    int alias = -1;        // output: index of the host input whose staging it shares
    bool scratch = false;  // output with a device slot only (written, never copied back)
    char* dup_dst = nullptr;  // scratch output copied host-side from output args[dup_of]
    int dup_of = -1;
    // assigned by staged():
    bool pinned = false;
    size_t dev_off = 0, pin_off = 0;  // byte offsets of the plane in a slot, per chunk element
    bool has_pin = false;
};

// Pieces of at most 8 MiB, so the pool's threads share one plane's copy.
void add_pieces(std::vector<Piece>& v, char* dst, const char* src, size_t bytes) {
    constexpr size_t kPiece = size_t(8) << 20;
    for (size_t at = 0; at < bytes; at += kPiece)
        v.push_back({dst + at, src + at, std::min(kPiece, bytes - at)});
}

// One direction's copies of a chunk, issued together after the loop that
// collects them (one cudaMemcpyAsync each).
struct CopyBatch {
    std::vector<void*> dst, src;
    std::vector<size_t> bytes;
    void add(void* d, const void* s, size_t b) {
        dst.push_back(d);
        src.push_back(const_cast<void*>(s));
        bytes.push_back(b);
    }
    fvb_status flush(cudaMemcpyKind kind, cudaStream_t s) {
        for (size_t i = 0; i < dst.size(); ++i) {
            const cudaError_t e = cudaMemcpyAsync(dst[i], src[i], bytes[i], kind, s);
            if (e != cudaSuccess)
                return cuda_fail(e, kind == cudaMemcpyHostToDevice ? "host->device copy"
                                                                   : "device->host copy");
        }
        dst.clear();
        src.clear();
        bytes.clear();
        return FVB_OK;
    }
};

// Copies between a slot's device staging and its pinned bounce buffer, one
// per run of planes that sit back to back in both layouts (in a pageable
// call usually all inputs in one run and all outputs in another) instead of
// one per plane: a small chunk costs a few microseconds per copy call.  A run
// also moves the unused tails of its inner planes (chunk - cnt elements),
// which stay inside both buffers and are never read.
struct BounceRuns {
    struct Run {
        size_t dev0, pin0, dev1, pin1, last_width;  // offsets in bytes per point
    };
    std::vector<Run> v;
    void add(size_t dev_off, size_t pin_off, size_t width) {
        if (!v.empty() && v.back().dev1 == dev_off && v.back().pin1 == pin_off) {
            v.back().dev1 += width;
            v.back().pin1 += width;
            v.back().last_width = width;
            return;
        }
        v.push_back({dev_off, pin_off, dev_off + width, pin_off + width, width});
    }
    void flush(char* dbase, char* pin, uint64_t chunk, uint64_t cnt, cudaMemcpyKind kind,
               CopyBatch& out) {
        for (const Run& r : v) {
            const size_t bytes = (r.dev1 - r.last_width - r.dev0) * chunk + cnt * r.last_width;
            char* d = dbase + r.dev0 * chunk;
            char* h = pin + r.pin0 * chunk;
            if (kind == cudaMemcpyHostToDevice)
                out.add(d, h, bytes);
            else
                out.add(h, d, bytes);
        }
        v.clear();
    }
};

// The staged executor.  `launch(dev_args, cnt, stream)` enqueues the kernel
// for one chunk; dev_args follow `args` (device pointers at the chunk, NULL
// for NULL slots).  Returns once every output is in place.
template <class Launch>
fvb_status staged(fvb_ctx* ctx, std::vector<Arg>& args, uint64_t n, Launch&& launch) {
    // staging layout: inputs first, then outputs not sharing an input's slot
    size_t dev_bpp = 0, pin_bpp = 0;
    bool any_pageable = false;
    for (Arg& a : args) {
        if (a.scratch) {
            a.dev_off = dev_bpp;
            dev_bpp += a.width;
            continue;
        }
        if (!a.host) continue;
        const Mem kind = memory_kind(a.host);
        if (kind == Mem::kDevice) return fail(FVB_EARG, "a host plane is device memory");
        a.pinned = kind == Mem::kPinned;
        if (a.out && a.alias >= 0) continue;
        a.dev_off = dev_bpp;
        dev_bpp += a.width;
        if (!a.pinned) {
            a.has_pin = true;
            a.pin_off = pin_bpp;
            pin_bpp += a.width;
            any_pageable = true;
        }
    }
    for (Arg& a : args)
        if (a.host && a.out && a.alias >= 0) {
            const Arg& src = args[size_t(a.alias)];
            a.dev_off = src.dev_off;
            a.pin_off = src.pin_off;
            a.has_pin = !a.pinned;
            if (a.has_pin && !src.has_pin) {  // pageable output over a pinned input: own bounce
                a.pin_off = pin_bpp;
                pin_bpp += a.width;
                any_pageable = true;
            }
        }
    // FVB_HOST_BOUNCE=0 disables the bounce buffers (tests of the fallback)
    static const bool allow_bounce = [] {
        const char* e = std::getenv("FVB_HOST_BOUNCE");
        return !(e && e[0] == '0' && e[1] == '\0');
    }();
    if (!allow_bounce) pin_bpp = 0;
    const uint64_t chunk = chunk_for(ctx, std::max<size_t>(dev_bpp, 1), n);
    bool bounce = allow_bounce;
    bool got_pinned = true;
    if (fvb_status st =
            ensure_buffers(ctx, size_t(chunk) * dev_bpp, size_t(chunk) * pin_bpp, &got_pinned))
        return st;
    bounce = bounce && got_pinned;
    if (!bounce) {  // no pinned memory: pageable planes go through cudaMemcpyAsync as they are
        for (Arg& a : args) a.has_pin = false;
        any_pageable = false;
    }
    bool any_dup = false;
    for (const Arg& a : args) any_dup |= a.dup_of >= 0;
    if ((any_pageable || any_dup) && !ctx->pool) {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        static const int knob = env_knob("FVB_POOL_THREADS", 0);
        const unsigned workers = knob > 0 ? unsigned(knob) : std::min(16u, hw) - 1;
        ctx->pool.reset(new (std::nothrow) CopyPool(workers));
    }
    auto copy = [&](const std::vector<Piece>& p) {
        if (ctx->pool)
            ctx->pool->run(p);
        else
            for (const Piece& q : p) host_copy(q.dst, q.src, q.bytes);
    };

    // On every exit -- an error part-way included -- nothing this call
    // enqueued may still be copying into or out of the caller's buffers.
    struct Drain {
        fvb_ctx* ctx;
        ~Drain() {
            for (int s = 0; s < ctx->slots; ++s) cudaStreamSynchronize(ctx->stream[s]);
        }
    } drain{ctx};
    const uint64_t nchunks = (n + chunk - 1) / chunk;
    int64_t pending[fvb_ctx::kMaxSlots];
    for (auto& p : pending) p = -1;
    std::vector<Piece> pieces;
    // Unpack the pageable outputs of the chunk a slot last carried.
    auto finish = [&](int slot) -> fvb_status {
        if (pending[slot] < 0) return FVB_OK;
        const uint64_t off = uint64_t(pending[slot]) * chunk;
        const uint64_t cnt = std::min(chunk, n - off);
        pending[slot] = -1;
        const cudaError_t e = cudaEventSynchronize(ctx->done[slot]);
        if (e != cudaSuccess) return cuda_fail(e, "pipeline chunk");
        pieces.clear();
        char* pin = static_cast<char*>(ctx->pin_buf[slot]);
        for (const Arg& a : args)
            if (a.out && a.host && a.has_pin)
                add_pieces(pieces, a.host + off * a.width, pin + a.pin_off * chunk, cnt * a.width);
        copy(pieces);
        if (any_dup) {  // duplicate outputs: from their (now complete) source output
            pieces.clear();
            for (const Arg& a : args)
                if (a.dup_of >= 0)
                    add_pieces(pieces, a.dup_dst + off * a.width,
                               args[size_t(a.dup_of)].host + off * a.width, cnt * a.width);
            copy(pieces);
        }
        return FVB_OK;
    };

    std::vector<void*> dargs(args.size());
    BounceRuns runs;
    CopyBatch copies;
    for (uint64_t c = 0; c < nchunks; ++c) {
        const int slot = int(c % ctx->slots);
        cudaStream_t s = ctx->stream[slot];
        const uint64_t off = c * chunk;
        const uint64_t cnt = std::min(chunk, n - off);
        char* dbase = static_cast<char*>(ctx->slot_buf[slot]);
        char* pin = static_cast<char*>(ctx->pin_buf[slot]);
        if (fvb_status st = finish(slot)) return st;  // the bounce buffers are free again
        // pack this chunk's pageable inputs
        pieces.clear();
        for (const Arg& a : args)
            if (!a.out && a.host && a.has_pin)
                add_pieces(pieces, pin + a.pin_off * chunk, a.host + off * a.width, cnt * a.width);
        // the slot's bounce buffer is then busy until this chunk's copies
        // complete: the next chunk on this slot must wait for them even when
        // no output is unpacked from it
        const bool packed = !pieces.empty();
        copy(pieces);
        for (size_t i = 0; i < args.size(); ++i) {
            const Arg& a = args[i];
            if (a.dev) {
                dargs[i] = a.dev + off * a.width;
                continue;
            }
            if (a.scratch) {
                dargs[i] = dbase + a.dev_off * chunk;
                continue;
            }
            if (!a.host) {
                dargs[i] = nullptr;
                continue;
            }
            dargs[i] = dbase + a.dev_off * chunk;
            if (a.out) continue;
            if (a.has_pin) {
                runs.add(a.dev_off, a.pin_off, a.width);
                continue;
            }
            if (a.pinned) {
                copies.add(dargs[i], a.host + off * a.width, cnt * a.width);
                continue;
            }
            // pageable without bounce buffers: the driver stages it
            const cudaError_t e = cudaMemcpyAsync(dargs[i], a.host + off * a.width,
                                                  cnt * a.width, cudaMemcpyHostToDevice, s);
            if (e != cudaSuccess) return cuda_fail(e, "host->device copy");
        }
        runs.flush(dbase, pin, chunk, cnt, cudaMemcpyHostToDevice, copies);
        if (fvb_status st = copies.flush(cudaMemcpyHostToDevice, s)) return st;
        if (fvb_status st = launch(dargs.data(), cnt, s)) return st;
        bool unpack = false;
        for (size_t i = 0; i < args.size(); ++i) {
            const Arg& a = args[i];
            if (!a.out || !a.host) continue;
            unpack |= a.has_pin;
            if (a.has_pin) {
                runs.add(a.dev_off, a.pin_off, a.width);
                continue;
            }
            if (a.pinned) {
                copies.add(a.host + off * a.width, dargs[i], cnt * a.width);
                continue;
            }
            const cudaError_t e = cudaMemcpyAsync(a.host + off * a.width, dargs[i], cnt * a.width,
                                                  cudaMemcpyDeviceToHost, s);
            if (e != cudaSuccess) return cuda_fail(e, "device->host copy");
        }
        runs.flush(dbase, pin, chunk, cnt, cudaMemcpyDeviceToHost, copies);
        if (fvb_status st = copies.flush(cudaMemcpyDeviceToHost, s)) return st;
        if (unpack || any_dup || packed) {
            const cudaError_t e = cudaEventRecord(ctx->done[slot], s);
            if (e != cudaSuccess) return cuda_fail(e, "chunk event");
            pending[slot] = int64_t(c);
        }
    }
    for (uint64_t c = nchunks > ctx->slots ? nchunks - ctx->slots : 0; c < nchunks; ++c)
        if (fvb_status st = finish(int(c % ctx->slots))) return st;
    for (int s = 0; s < ctx->slots; ++s) {
        const cudaError_t e = cudaStreamSynchronize(ctx->stream[s]);
        if (e != cudaSuccess) return cuda_fail(e, "pipeline completion");
    }
    return FVB_OK;
}

// Host-side outputs, written by host threads concurrently with the device
// pipeline instead of crossing PCIe:
//  - pass-through items: output j < PASS is bit-for-bit input plane 1 + j
//    (the flux's row 0 is the momentum fields themselves,
//    include/fusevec/fluid.hpp:168-169); the host already holds those bytes;
//  - constant items (the Jacobian's 0 / 1 / gamma-1 entries, 30 of 75 in
//    3-D): every element is the same value of T, filled in place.
// (Duplicate items -- JacobianOp::duplicate_of, 18 of 75 -- are copied
// host-side too, but per chunk, once their source output has landed: the
// staged executor's dup_of.)
// Joined on every exit path.
struct HostJob {
    char* dst;
    const char* src;  // nullptr: fill with `fill` (the bits of one T)
    uint64_t fill;
};

template <class T>
struct HostSide {
    std::vector<std::thread> workers;
    HostSide(const std::vector<HostJob>& jobs, size_t bytes) {
        if (jobs.empty() || bytes == 0) return;
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const size_t total = jobs.size() * bytes;
        // Four threads by default (a quarter of a 16-core host): more copy
        // threads slow the concurrent DMA into host memory more than they
        // gain (A/B on two boxes, profiles/r02_e2e_fill_threads_ab.jsonl:
        // 8 threads cost the flux e2e 2.4-3.4% and the Jacobian's 2-5%).
        // At most one thread per MiB: starting and joining one costs tens of
        // microseconds, so a small call writes inline (below).
        static const int knob = env_knob("FVB_FILL_THREADS", 0);
        const unsigned cap = knob > 0 ? unsigned(knob) : std::min(4u, std::max(2u, hw / 4));
        const unsigned nt = unsigned(std::min<size_t>(cap,
                                                      std::max<size_t>(1, total >> 20)));
        const size_t per = ((total + nt - 1) / nt + 63) & ~size_t(63);  // whole elements
        auto work = [jobs, bytes](size_t lo, size_t hi) {
            while (lo < hi) {
                const HostJob& j = jobs[lo / bytes];
                const size_t at = lo % bytes;
                const size_t len = std::min(hi - lo, bytes - at);
                if (j.src)
                    host_copy(j.dst + at, j.src + at, len);
                else
                    host_fill(j.dst + at, j.fill, sizeof(T), len);
                lo += len;
            }
        };
        if (nt == 1) {
            work(0, total);
            return;
        }
        try {
            for (unsigned t = 0; t < nt && size_t(t) * per < total; ++t) {
                const size_t lo = size_t(t) * per;
                workers.emplace_back(work, lo, std::min(total, lo + per));
            }
        } catch (...) {  // no threads to be had: on the calling thread
            for (auto& w : workers) w.join();
            workers.clear();
            work(0, total);
        }
    }
    ~HostSide() {
        for (auto& w : workers) w.join();
    }
};

fvb_status reset_lambda(fvb_ctx* ctx, size_t bytes) {
    cudaError_t e = cudaMemsetAsync(ctx->red, 0, bytes, ctx->stream[0]);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->reset_done, ctx->stream[0]);
    for (int s = 1; s < ctx->slots && e == cudaSuccess; ++s)
        e = cudaStreamWaitEvent(ctx->stream[s], ctx->reset_done, 0);
    return e == cudaSuccess ? FVB_OK : cuda_fail(e, "lambda reset");
}

template <class T>
fvb_status read_lambda(fvb_ctx* ctx, double* lambda_max) {
    using Bu = typename Bits<T>::U;
    Bu bits = 0;
    const cudaError_t e = cudaMemcpy(&bits, ctx->red, sizeof(Bu), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "lambda_max read-back");
    T v;
    std::memcpy(&v, &bits, sizeof v);
    *lambda_max = double(v);
    return FVB_OK;
}

template <class Op, class T, bool RED, bool TUNE, int PASS = 0, bool FILL = false>
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
    if (PASS > 0 || FILL) {  // host threads write some outputs while the pipeline writes others
        std::vector<uintptr_t> starts;
        for (int j = 0; j < NOUT; ++j) starts.push_back(reinterpret_cast<uintptr_t>(out[j]));
        std::sort(starts.begin(), starts.end());
        if (std::adjacent_find(starts.begin(), starts.end()) != starts.end())
            return fail(FVB_EARG, "two host outputs name one plane");
    }
    DeviceGuard guard(ctx->device);
    if (fvb_status st = host_planes(in, NIN, sizeof(T))) return st;
    if (fvb_status st = host_planes(const_cast<const void* const*>(out), NOUT, sizeof(T)))
        return st;
    using Bu = typename Bits<T>::U;
    if (RED)
        if (fvb_status st = reset_lambda(ctx, sizeof(Bu))) return st;
    if (n == 0) {
        if (RED && lambda_max) *lambda_max = 0.0;
        return FVB_OK;
    }
    std::vector<Arg> args;
    for (int i = 0; i < NIN; ++i)
        args.push_back({static_cast<char*>(const_cast<void*>(in[i])), nullptr, sizeof(T), false});
    std::vector<HostJob> host_side;
    for (int j = 0; j < NOUT; ++j) {
        // pass-through and constant outputs are written host-side; the
        // kernel's copy of them lands in a device scratch slot
        bool on_host = j < PASS;
        if (on_host) {
            host_side.push_back({static_cast<char*>(out[j]),
                                 static_cast<const char*>(in[1 + j]), 0});
        }
        int dup = -1;
        if constexpr (FILL) {
            T v;
            if (!on_host && Op::constant_item(j, k, &v)) {
                uint64_t bits = 0;
                std::memcpy(&bits, &v, sizeof v);
                host_side.push_back({static_cast<char*>(out[j]), nullptr, bits});
                on_host = true;
            } else if (!on_host) {
                static const bool dups_on_link = env_knob("FVB_DUPS_ON_LINK", 0) != 0;
                if (!dups_on_link)
                    dup = Op::duplicate_of(j);  // an earlier, computed and shipped output
            }
        }
        Arg a{on_host || dup >= 0 ? nullptr : static_cast<char*>(out[j]), nullptr, sizeof(T), true};
        a.scratch = on_host || dup >= 0;
        if (dup >= 0) {
            a.dup_dst = static_cast<char*>(out[j]);
            a.dup_of = NIN + dup;
        }
        args.push_back(a);
    }
    HostSide<T> host_writes(host_side, size_t(n) * sizeof(T));
    fvb_status st = staged(ctx, args, n, [&](void* const* d, uint64_t cnt, cudaStream_t s) {
        const T* din[NIN];
        T* dout[NOUT > 0 ? NOUT : 1];
        for (int i = 0; i < NIN; ++i) din[i] = static_cast<const T*>(d[i]);
        for (int j = 0; j < NOUT; ++j) dout[j] = static_cast<T*>(d[NIN + j]);
        return launch_op<Op, T, RED, TUNE>(din, dout, cnt, k, static_cast<Bu*>(ctx->red), s);
    });
    if (st) return st;
    if (RED && lambda_max) return read_lambda<T>(ctx, lambda_max);
    return FVB_OK;
}

// PASS_DIM: the first d outputs are pass-through copies of inputs 1..d.
// FILL: outputs the op reports as constant items are filled host-side.
template <template <class, int> class OpT, bool RED, class T, bool TUNE3 = false,
          bool PASS_DIM = false, bool FILL = false>
fvb_status pipeline_dim(fvb_ctx* ctx, const fvb_gas* gas, uint32_t dim, const void* const* in,
                        void* const* out, uint64_t n, double* lambda_max) {
    const auto k = make_consts<T>(gas);
    switch (dim) {
        case 1:
            return pipeline<OpT<T, 1>, T, RED, false, PASS_DIM ? 1 : 0, FILL>(ctx, in, out, n, k,
                                                                              lambda_max);
        case 2:
            return pipeline<OpT<T, 2>, T, RED, false, PASS_DIM ? 2 : 0, FILL>(ctx, in, out, n, k,
                                                                              lambda_max);
        default:
            return pipeline<OpT<T, 3>, T, RED, TUNE3, PASS_DIM ? 3 : 0, FILL>(ctx, in, out, n, k,
                                                                              lambda_max);
    }
}

// fvb_launch_host with a hand-written Jacobian kernel (the reference's
// Jacobian block through the adapter or the JIT seam): the same host-side
// treatment as fvb_jacobian_host -- constant entries filled by host threads,
// duplicate entries shipped once and copied per chunk -- for host output
// slots that alias no input.  Both are exactly what the kernel would write
// (its own Consts, JacobianOp's own item tables).
template <class T, int D>
void jacobian_host_side(const fvb_kernel* k, std::vector<Arg>& v, std::vector<HostJob>& fills) {
    using Op = JacobianOp<T, D>;
    if (k->n_outputs != uint32_t(Op::NOUT)) return;
    const Consts<T> c{static_cast<T>(k->consts[0]), static_cast<T>(k->consts[1]),
                      static_cast<T>(k->consts[2]), static_cast<T>(k->consts[3]),
                      static_cast<T>(k->consts[4]), static_cast<T>(k->consts[5])};
    for (int j = 0; j < Op::NOUT; ++j) {
        Arg& a = v[size_t(j)];
        if (!a.host || a.alias >= 0 || a.width != sizeof(T)) continue;
        T val;
        if (Op::constant_item(j, c, &val)) {
            uint64_t bits = 0;
            std::memcpy(&bits, &val, sizeof val);
            fills.push_back({a.host, nullptr, bits});
            a.host = nullptr;
            a.scratch = true;
            continue;
        }
        const int d = Op::duplicate_of(j);
        if (d < 0) continue;
        const Arg& src = v[size_t(d)];
        if (!src.host || src.alias >= 0 || src.dup_of >= 0 || src.width != sizeof(T)) continue;
        a.dup_dst = a.host;
        a.dup_of = d;
        a.host = nullptr;
        a.scratch = true;
    }
}

void launch_host_side(const fvb_kernel* k, std::vector<Arg>& v, std::vector<HostJob>& fills) {
    if (k->impl || std::strncmp(k->name, "jacobian", 8) != 0) return;
    switch (k->dim * 2 + k->prec) {
        case 2: return jacobian_host_side<float, 1>(k, v, fills);
        case 3: return jacobian_host_side<double, 1>(k, v, fills);
        case 4: return jacobian_host_side<float, 2>(k, v, fills);
        case 5: return jacobian_host_side<double, 2>(k, v, fills);
        case 6: return jacobian_host_side<float, 3>(k, v, fills);
        case 7: return jacobian_host_side<double, 3>(k, v, fills);
        default: return;
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
    static const int slots = env_knob("FVB_HOST_SLOTS", 3);
    ctx->slots = std::min(fvb_ctx::kMaxSlots, std::max(2, slots));
    DeviceGuard guard(device);
    for (int s = 0; s < ctx->slots && e == cudaSuccess; ++s) {
        e = cudaStreamCreateWithFlags(&ctx->stream[s], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->done[s], cudaEventDisableTiming);
    }
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
    for (int s = 0; s < ctx->slots; ++s) {
        if (ctx->stream[s]) cudaStreamSynchronize(ctx->stream[s]);
        if (ctx->slot_buf[s]) cudaFree(ctx->slot_buf[s]);
        if (ctx->pin_buf[s]) cudaFreeHost(ctx->pin_buf[s]);
        if (ctx->done[s]) cudaEventDestroy(ctx->done[s]);
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
        // the constant entries are filled host-side (JacobianOp::constant_item)
        if (prec == FVB_F64) {
            if (lambda_max)
                return pipeline_dim<JacobianOp, true, double, false, false, true>(
                    ctx, gas, dim, in, out, n, lambda_max);
            return pipeline_dim<JacobianOp, false, double, false, false, true>(ctx, gas, dim, in,
                                                                              out, n, nullptr);
        }
        if (lambda_max)
            return pipeline_dim<JacobianOp, true, float, false, false, true>(ctx, gas, dim, in,
                                                                            out, n, lambda_max);
        return pipeline_dim<JacobianOp, false, float, false, false, true>(ctx, gas, dim, in, out,
                                                                         n, nullptr);
    });
}

fvb_status fvb_launch_host(fvb_ctx* ctx, const fvb_kernel* k, uint64_t n, void* const* args,
                           const uint8_t* arg_prec, const uint8_t* arg_on_device,
                           double* lambda_max, void* after) {
    return guarded([&]() -> fvb_status {
        if (!ctx || !k || !args || !arg_prec) return fail(FVB_EARG, "NULL argument");
        if (lambda_max && !k->reduce) return fail(FVB_EARG, "kernel has no CFL reduction");
        const size_t nargs = size_t(k->n_outputs) + k->n_inputs;
        if (nargs == 0) return fail(FVB_EARG, "kernel without arguments");
        std::vector<Arg> v(nargs);
        for (size_t i = 0; i < nargs; ++i) {
            if (arg_prec[i] > 1) return fail(FVB_EPREC, "argument precision must be 0 or 1");
            Arg& a = v[i];
            a.width = arg_prec[i] ? 8 : 4;
            a.out = i < k->n_outputs;
            const uint8_t where = arg_on_device ? arg_on_device[i] : 0;
            if (where == 2) {  // written on the device, never copied back
                if (!a.out) return fail(FVB_EARG, "only an output slot can be discarded");
                a.scratch = true;
                continue;
            }
            if (!args[i]) {
                if (!a.out) return fail(FVB_EARG, "NULL leaf plane");
                continue;  // a NULL output slot (e.g. reduce-only wave speed)
            }
            if (where) {
                a.dev = static_cast<char*>(args[i]);
            } else {
                a.host = static_cast<char*>(args[i]);
            }
        }
        // In place: an output that is a host leaf shares its staging; any
        // other overlap between host planes has no element-wise meaning.
        for (size_t j = 0; j < k->n_outputs; ++j) {
            Arg& o = v[j];
            if (!o.host) continue;
            const uintptr_t olo = uintptr_t(o.host), ohi = olo + n * o.width;
            for (size_t i = 0; i < nargs; ++i) {
                if (i == j || !v[i].host) continue;
                const uintptr_t lo = uintptr_t(v[i].host), hi = lo + n * v[i].width;
                if (lo == olo && v[i].width == o.width) {
                    if (i >= k->n_outputs && o.alias < 0) o.alias = int(i);
                    else if (i < k->n_outputs)
                        return fail(FVB_EARG, "two host outputs name one plane");
                } else if (lo < ohi && olo < hi && n > 0) {
                    return fail(FVB_EARG, "host planes overlap at an offset");
                }
            }
        }
        DeviceGuard guard(ctx->device);
        for (const Arg& a : v)
            if (fvb_status st =
                    host_planes(reinterpret_cast<const void* const*>(&a.host), 1, a.width))
                return st;
        const size_t red_bytes = k->prec ? 8 : 4;  // the kernel's accumulator
        if (lambda_max)
            if (fvb_status st = reset_lambda(ctx, red_bytes)) return st;
        if (after) {  // device work the caller queued first (producing resident planes)
            cudaError_t e = cudaEventRecord(ctx->reset_done, static_cast<cudaStream_t>(after));
            for (int s = 0; s < ctx->slots && e == cudaSuccess; ++s)
                e = cudaStreamWaitEvent(ctx->stream[s], ctx->reset_done, 0);
            if (e != cudaSuccess) return cuda_fail(e, "ordering after the caller's stream");
        }
        if (n == 0) {
            if (lambda_max) *lambda_max = 0.0;
            return FVB_OK;
        }
        std::vector<HostJob> fills;
        launch_host_side(k, v, fills);
        fvb_status st;
        {
            // fills run on host threads while the pipeline streams; joined
            // (on every exit) before the call returns
            HostSide<double> fill_d(k->prec ? fills : std::vector<HostJob>{}, n * 8);
            HostSide<float> fill_f(k->prec ? std::vector<HostJob>{} : fills, n * 4);
            st = staged(ctx, v, n, [&](void* const* d, uint64_t cnt, cudaStream_t s) {
                if (lambda_max) return k->reduce(k, 0, cnt, d, ctx->red, s);
                return k->fn(k, 0, cnt, d, s);
            });
        }
        if (st) return st;
        if (lambda_max) return red_bytes == 8 ? read_lambda<double>(ctx, lambda_max)
                                              : read_lambda<float>(ctx, lambda_max);
        return FVB_OK;
    });
}

}  // extern "C"
