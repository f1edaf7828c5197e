// fusevec_device.cpp -- see fusevec_device.hpp.
//
// Compiled against the reference's public headers (the maintainer's
// fusevec, or in our tests the reference built as namespace fvref), linked
// with libfvb.so and the CUDA runtime.
#include "fusevec_device.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>

#include "fvb.h"

namespace fusevec {

// ---------------------------------------------------------------------------
// New fluid expression objects, built only from the public Expr API in the
// style of proj/src/fluid.cpp (SURVEY Appendix A gives the operation order;
// the fused kernels and the registry patterns mirror exactly these trees).
// ---------------------------------------------------------------------------

namespace {

double gm1_of(const EosSpec& eos) { return (eos.R() / eos.cv()).value(); }

void require_conservative(const StateSet& u, const char* what) {
    if (u.formulation() != Formulation::Conservative)
        throw BadMap(std::string(what) + " needs a conservative state");
}

}  // namespace

Expr derived_c(const StateSet& u) {
    // A.2: elem_sqrt((constant(gamma, p) * p) / rho)
    Expr p = derived_p(u);
    const Expr& rho = u.field(VarKind::Density);
    return elem_sqrt((constant(u.eos().gamma_value(), p) * p) / rho);
}

Expr wave_speed(const StateSet& u) {
    // A.4: elem_sqrt(derived_v_mag2(u)) + c
    require_conservative(u, "wave_speed");
    return elem_sqrt(derived_v_mag2(u)) + derived_c(u);
}

BlockExpr inviscid_flux_jacobian(const StateSet& u) {
    // A.3, items [k][r][c] of a (d*(d+2)) x (d+2) row-major block.
    require_conservative(u, "inviscid_flux_jacobian");
    const std::size_t d = u.dim(), w = d + 2;
    const Expr& rho = u.field(VarKind::Density);
    const Expr& rho_E = u.field(VarKind::TotalEnergy);
    Expr p = derived_p(u);
    std::vector<Expr> v(d);
    for (std::size_t j = 0; j < d; ++j) v[j] = u.field(1 + j) / rho;
    Expr q2;
    for (std::size_t j = 0; j < d; ++j) q2 = q2.valid() ? q2 + v[j] * v[j] : v[j] * v[j];
    Expr H = (rho_E + p) / rho;
    const double gm1 = gm1_of(u.eos());
    Expr phi = constant(0.5, q2) * (constant(gm1, q2) * q2);
    auto lit = [&](double x) { return constant(x, rho); };

    std::vector<BlockItem> items;
    items.reserve(d * w * w);
    for (std::size_t k = 0; k < d; ++k) {
        for (std::size_t c = 0; c < w; ++c) items.push_back(BlockItem(lit(c == 1 + k ? 1.0 : 0.0)));
        for (std::size_t i = 0; i < d; ++i) {
            items.push_back(BlockItem(i == k ? phi - v[i] * v[k] : -(v[i] * v[k])));
            for (std::size_t j = 0; j < d; ++j) {
                Expr acc;
                if (i == j) acc = v[k];
                if (j == k) acc = acc.valid() ? acc + v[i] : v[i];
                if (i == k) {
                    Expr t = -(constant(gm1, v[j]) * v[j]);
                    acc = acc.valid() ? acc + t : t;
                }
                items.push_back(BlockItem(acc.valid() ? acc : lit(0.0)));
            }
            items.push_back(BlockItem(lit(i == k ? gm1 : 0.0)));
        }
        items.push_back(BlockItem(v[k] * (phi - H)));
        for (std::size_t j = 0; j < d; ++j) {
            Expr ujuk = v[j] * v[k];
            items.push_back(BlockItem(j == k ? H - constant(gm1, ujuk) * ujuk
                                             : -(constant(gm1, ujuk) * ujuk)));
        }
        items.push_back(BlockItem(constant(u.eos().gamma_value(), v[k]) * v[k]));
    }
    return BlockExpr(d * w, w, std::move(items));
}

namespace device {

namespace {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw DeviceError(std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                          cudaGetErrorString(e) + ")");
}

void fvb_check(fvb_status st) {
    if (st == FVB_OK) return;
    std::string msg = fvb_last_error();
    switch (st) {
        case FVB_ELEN: throw LengthMismatch(msg);
        case FVB_EUNSUPPORTED: throw UnsupportedExpression(msg);
        case FVB_ECUDA: throw DeviceError(msg);
        default: throw Error(msg);
    }
}

char prec_char(Precision p) { return p == Precision::f32 ? 's' : 'd'; }

double narrow(double v, Precision p) {
    return p == Precision::f32 ? static_cast<double>(static_cast<float>(v)) : v;
}

// Leaf slots across one key: distinct DenseVectors in first-appearance
// left-to-right DFS order (proj/src/backend_jit.cpp:78-99).
struct Slots {
    std::vector<const DenseVector*> v;
    std::size_t of(const DenseVector* x) {
        for (std::size_t i = 0; i < v.size(); ++i)
            if (v[i] == x) return i;
        v.push_back(x);
        return v.size() - 1;
    }
};

// The key text is written through a raw cursor into a string grown ahead
// in large steps (a 75-item Jacobian key is ~4.4 KB, built on every
// evaluate_block call whose trees are not reused): no per-character
// capacity checks.
struct KeyOut {
    std::string& s;
    char* p;
    char* end;
    explicit KeyOut(std::string& str) : s(str) {
        const std::size_t used = s.size();
        s.resize(std::max<std::size_t>(used + 1024, 2 * used));
        p = &s[0] + used;
        end = &s[0] + s.size();
    }
    // the slow path, out of line: the string doubles
    __attribute__((noinline)) void grow(std::size_t k) {
        const std::size_t used = std::size_t(p - &s[0]);
        s.resize(std::max(2 * s.size(), used + k + 1024));
        p = &s[0] + used;
        end = &s[0] + s.size();
    }
    char* room(std::size_t k) {
        if (std::size_t(end - p) < k) grow(k);
        char* q = p;
        p += k;
        return q;
    }
    void put(char c) { *room(1) = c; }
    void uint(std::size_t v) {
        if (v < 10) {
            put(char('0' + v));
            return;
        }
        char buf[24];
        int i = 0;
        do {
            buf[i++] = char('0' + v % 10);
            v /= 10;
        } while (v);
        char* q = room(std::size_t(i));
        while (i) *q++ = buf[--i];
    }
    void hex16(unsigned long long bits) {
        static const char kHex[] = "0123456789abcdef";
        char* q = room(16);
        for (int i = 15; i >= 0; --i, bits >>= 4) q[i] = kHex[bits & 15];
    }
    void finish() { s.resize(std::size_t(p - &s[0])); }
};

// key_node (proj/src/backend_jit.cpp:112-155): same grammar, same order.
void key_node(const ExprNode& n, Slots& slots, bool& ok, KeyOut& out) {
    switch (n.kind) {
        case NodeKind::Leaf: {
            out.put('L');
            out.put(prec_char(n.prec));
            out.uint(slots.of(n.vec));
            out.put(';');
            return;
        }
        case NodeKind::Constant: {
            const double v = narrow(n.value, n.prec);
            if (!std::isfinite(v)) ok = false;
            unsigned long long bits;
            std::memcpy(&bits, &v, sizeof bits);
            out.put('C');
            out.put(prec_char(n.prec));
            out.hex16(bits);
            out.put(';');
            return;
        }
        case NodeKind::Tagged:
        case NodeKind::Cached:
            key_node(*n.left, slots, ok, out);
            return;
        case NodeKind::Unary:
            out.put('U');
            out.uint(static_cast<std::size_t>(n.uop));
            out.put(prec_char(n.prec));
            out.put('(');
            key_node(*n.left, slots, ok, out);
            out.put(')');
            return;
        case NodeKind::Binary:
            out.put('B');
            out.uint(static_cast<std::size_t>(n.bop));
            out.put(prec_char(n.prec));
            out.put('(');
            key_node(*n.left, slots, ok, out);
            out.put(',');
            key_node(*n.right, slots, ok, out);
            out.put(')');
            return;
    }
}

void key_node(const ExprNode& n, Slots& slots, bool& ok, std::string& out) {
    KeyOut w(out);
    key_node(n, slots, ok, w);
    w.finish();
}

// validate() semantics of proj/src/backend_eval.cpp:236-265.
void validate(const ExprNode& n, std::size_t len, std::map<int, const DenseVector*>& tags) {
    switch (n.kind) {
        case NodeKind::Leaf:
            if (n.vec->size() != len)
                throw LengthMismatch("leaf length " + std::to_string(n.vec->size()) +
                                     " does not match destination length " + std::to_string(len));
            return;
        case NodeKind::Constant:
            return;
        case NodeKind::Tagged:
            if (n.left->kind == NodeKind::Leaf) {
                auto [it, inserted] = tags.emplace(n.tag, n.left->vec);
                if (!inserted && it->second != n.left->vec)
                    throw TagConflict("tag " + std::to_string(n.tag) +
                                      " bound to two different leaves");
            }
            validate(*n.left, len, tags);
            return;
        case NodeKind::Cached:
        case NodeKind::Unary:
            validate(*n.left, len, tags);
            return;
        case NodeKind::Binary:
            validate(*n.left, len, tags);
            validate(*n.right, len, tags);
            return;
    }
}

const DenseVector* bare_leaf(const ExprNode& n) {
    if (n.kind == NodeKind::Leaf) return n.vec;
    if (n.kind == NodeKind::Tagged || n.kind == NodeKind::Cached) return bare_leaf(*n.left);
    return nullptr;
}

// A bare constant item (e.g. the Jacobian's 0 / 1 / gamma-1 entries): the
// bits every element of a destination of precision `dest` holds once the
// reference evaluates it -- the constant narrowed to its own precision
// (narrow_value, proj/src/scalar_ops.hpp:81-85), then stored as `dest`.
bool bare_constant(const ExprNode& n, Precision dest, uint64_t* bits) {
    if (n.kind == NodeKind::Tagged || n.kind == NodeKind::Cached)
        return bare_constant(*n.left, dest, bits);
    if (n.kind != NodeKind::Constant) return false;
    const double v = n.prec == Precision::f32 ? double(float(n.value)) : n.value;
    *bits = 0;
    if (dest == Precision::f32) {
        const float f = float(v);
        std::memcpy(bits, &f, sizeof f);
    } else {
        std::memcpy(bits, &v, sizeof v);
    }
    return true;
}

// One output of a plan: a host vector (staged), a device plane, or neither
// (a NULL slot: the reduce-only wave-speed pass writes no plane).
struct Out {
    DenseVector* host = nullptr;
    DeviceVector* dev = nullptr;
    Precision null_prec = Precision::f64;
    std::size_t null_size = 0;
    bool is_null() const { return !host && !dev; }
    Precision prec() const {
        return host ? host->precision() : dev ? dev->precision() : null_prec;
    }
    std::size_t size() const { return host ? host->size() : dev ? dev->size() : null_size; }
};

struct Plan {
    fvb_kernel k{};
    std::vector<const DenseVector*> leaves;
    std::vector<Out> outs;
    // Per output: the host leaf a bare-leaf item copies (the flux's row 0 is
    // the momentum fields), when that copy can be made host-side instead of
    // crossing PCIe twice; nullptr otherwise.  Set by block_impl.
    std::vector<const DenseVector*> pass_src;
    // Per output: 1 when a bare constant item is filled host-side (bits in
    // fill_bits) instead of shipped over PCIe.  Set by block_impl.
    std::vector<char> has_fill;
    std::vector<uint64_t> fill_bits;
};

// One host-side write: a copy of src, or (src == nullptr) a fill of every
// element of dst with the bits `fill` of dst's precision.
struct HostWrite {
    DenseVector* dst;
    const DenseVector* src;
    uint64_t fill;
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
        if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// The C library's host-buffer context for one device: staging slots, pinned
// bounce buffers for pageable DenseVectors and the copy threads
// (fvb_launch_host).  The reference's backends are re-entrant -- evaluate()
// may run on several host threads at once -- so staged evaluations on one
// device take turns on it (each is bound by the PCIe link anyway).
struct HostCtx {
    std::mutex mu;
    fvb_ctx* ctx = nullptr;
};

HostCtx& host_ctx(int ordinal) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<HostCtx>> per;
    std::lock_guard<std::mutex> lock(mu);
    auto& p = per[ordinal];
    if (!p) p = std::make_unique<HostCtx>();
    return *p;
}

// Host-side copies of pass-through items and fills of constant items, on a
// few threads, running while the device pipeline streams the computed
// items.  Joined on destruction.
struct HostCopies {
    std::vector<std::thread> threads;
    explicit HostCopies(const std::vector<HostWrite>& jobs) {
        if (jobs.empty()) return;
        std::size_t total = 0;
        for (const auto& j : jobs) total += j.dst->byte_size();
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        // a thread per 1 MiB at most (starting one costs tens of microseconds)
        const unsigned nt = unsigned(std::min<std::size_t>(std::min<unsigned>(4u, std::max(1u, hw / 4)),
                                                           std::max<std::size_t>(1, total >> 20)));
        const std::size_t per = ((total + nt - 1) / nt + 63) & ~std::size_t(63);  // whole elements
        auto copy = [jobs](std::size_t lo, std::size_t hi) {
            std::size_t base = 0;
            for (const HostWrite& j : jobs) {
                const std::size_t b = j.dst->byte_size();
                // the thread boundaries, rounded down to whole elements of
                // this job relative to its own start: neighbouring threads
                // round the shared boundary alike, so the pieces still tile
                // the job, and every piece starts element-aligned (jobs of
                // mixed precisions put f64 jobs at 4 mod 8 of the range)
                if (hi <= base || lo >= base + b) {
                    base += b;
                    continue;
                }
                const std::size_t w = j.dst->precision() == Precision::f64 ? 8 : 4;
                const std::size_t a = base + ((std::max(lo, base) - base) & ~(w - 1));
                const std::size_t e = base + ((std::min(hi, base + b) - base) & ~(w - 1));
                char* d = static_cast<char*>(j.dst->raw()) + (a - base);
                if (a < e && j.src) {
                    std::memcpy(d, static_cast<const char*>(j.src->raw()) + (a - base), e - a);
                } else if (a < e && j.fill == 0) {
                    std::memset(d, 0, e - a);
                } else if (a < e && j.dst->precision() == Precision::f64) {
                    double v;
                    std::memcpy(&v, &j.fill, sizeof v);
                    std::fill_n(reinterpret_cast<double*>(d), (e - a) / sizeof v, v);
                } else if (a < e) {
                    float v;
                    std::memcpy(&v, &j.fill, sizeof v);
                    std::fill_n(reinterpret_cast<float*>(d), (e - a) / sizeof v, v);
                }
                base += b;
            }
        };
        if (nt == 1) {
            copy(0, total);
            return;
        }
        try {
            for (unsigned t = 0; t < nt; ++t)
                threads.emplace_back(copy, std::size_t(t) * per, std::min(total, (t + 1) * per));
        } catch (...) {
            for (auto& th : threads) th.join();
            threads.clear();
            copy(0, total);
        }
    }
    ~HostCopies() {
        for (auto& th : threads) th.join();
    }
};

// The CFL maximum of several slices, combined the way the kernel combines
// points: IEEE bit patterns of the kernel's precision compared as unsigned
// integers (wave speeds are >= 0; a NaN anywhere wins).
double combine_max(const std::vector<double>& v, bool f64) {
    uint64_t best = 0;
    for (double x : v) {
        uint64_t b;
        if (f64) {
            std::memcpy(&b, &x, 8);
        } else {
            const float f = static_cast<float>(x);
            uint32_t u;
            std::memcpy(&u, &f, 4);
            b = u;
        }
        best = b > best ? b : best;
    }
    if (f64) {
        double d;
        std::memcpy(&d, &best, 8);
        return d;
    }
    const uint32_t u = static_cast<uint32_t>(best);
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// A host-buffer evaluation spread over DeviceBackend::ordinals: slice g of
// [0, n) runs on ordinal g through that device's host context, all slices at
// once on their own host threads (each device has its own PCIe link).
double run_sliced(const DeviceBackend& be, const Plan& plan, std::size_t n,
                  const std::vector<void*>& args, const std::vector<uint8_t>& prec,
                  const std::vector<uint8_t>& on_dev, bool reduce,
                  const std::vector<HostWrite>& pass) {
    const std::size_t G = be.ordinals.size();
    std::vector<double> lam(G, 0.0);
    std::vector<fvb_status> st(G, FVB_OK);
    std::vector<std::string> err(G);
    {
        HostCopies copies(pass);
        std::vector<std::thread> pool;
        for (std::size_t g = 0; g < G; ++g) {
            const std::size_t lo = n * g / G, hi = n * (g + 1) / G;
            if (hi == lo) continue;
            pool.emplace_back([&, g, lo, hi] {
                std::vector<void*> a(args);
                for (std::size_t i = 0; i < a.size(); ++i)
                    if (a[i] && on_dev[i] == 0) a[i] = static_cast<char*>(a[i]) + lo * (prec[i] ? 8 : 4);
                HostCtx& hc = host_ctx(be.ordinals[g]);
                std::lock_guard<std::mutex> lock(hc.mu);
                fvb_status s = FVB_OK;
                if (!hc.ctx) s = fvb_ctx_create(be.ordinals[g], be.chunk_points, &hc.ctx);
                if (s == FVB_OK)
                    s = fvb_launch_host(hc.ctx, &plan.k, hi - lo, a.data(), prec.data(),
                                        on_dev.data(), reduce ? &lam[g] : nullptr, nullptr);
                st[g] = s;
                if (s != FVB_OK) err[g] = fvb_last_error();
            });
        }
        for (auto& t : pool) t.join();
    }
    for (std::size_t g = 0; g < G; ++g)
        if (st[g] != FVB_OK) {
            const std::string msg = "device " + std::to_string(be.ordinals[g]) + ": " + err[g];
            switch (st[g]) {
                case FVB_ELEN: throw LengthMismatch(msg);
                case FVB_EUNSUPPORTED: throw UnsupportedExpression(msg);
                case FVB_ECUDA: throw DeviceError(msg);
                default: throw Error(msg);
            }
        }
    return reduce ? combine_max(lam, plan.k.prec != 0) : 0.0;
}

// Execute a plan over [0, n).  Device planes (resident leaves, device
// destinations) are used in place; with every plane on the device it is one
// launch on the backend's stream.  Otherwise fvb_launch_host streams the
// range through the device in chunks, DMA-ing pinned host planes directly
// and packing pageable ones through pinned bounce buffers.  With red !=
// nullptr (a device scalar of the kernel's precision, zeroed) the kernel's
// CFL reduction runs too and its result lands in *red.
void run(const DeviceBackend& be, Plan& plan, std::size_t n, void* red) {
    if (n == 0) return;
    DeviceGuard guard(be.ordinal);
    const std::size_t nout = plan.outs.size(), nin = plan.leaves.size();
    std::vector<void*> args(nout + nin, nullptr);
    std::vector<uint8_t> prec(nout + nin, 1), on_dev(nout + nin, 0);
    bool staged = false;
    std::vector<HostWrite> pass;
    for (std::size_t j = 0; j < nout; ++j) {
        const Out& o = plan.outs[j];
        prec[j] = o.prec() == Precision::f64 ? 1 : 0;
        if (j < plan.pass_src.size() && plan.pass_src[j]) {
            on_dev[j] = 2;  // computed into device scratch only; copied host-side
            pass.push_back({o.host, plan.pass_src[j], 0});
            staged = true;
        } else if (j < plan.has_fill.size() && plan.has_fill[j]) {
            on_dev[j] = 2;  // computed into device scratch only; filled host-side
            pass.push_back({o.host, nullptr, plan.fill_bits[j]});
            staged = true;
        } else if (o.dev) {
            args[j] = o.dev->data();
            on_dev[j] = 1;
        } else if (o.host) {
            args[j] = o.host->raw();
            staged = true;
        }
    }
    for (std::size_t i = 0; i < nin; ++i) {
        const DenseVector* l = plan.leaves[i];
        prec[nout + i] = l->precision() == Precision::f64 ? 1 : 0;
        if (DeviceVector* dv = be.residency ? be.residency->find(l) : nullptr) {
            if (dv->size() != n || dv->precision() != l->precision())
                throw LengthMismatch("resident plane does not match its host leaf");
            args[nout + i] = dv->data();
            on_dev[nout + i] = 1;
        } else {
            args[nout + i] = const_cast<void*>(static_cast<const void*>(l->raw()));
            staged = true;
        }
    }
    cudaStream_t s = static_cast<cudaStream_t>(be.stream);
    if (!staged) {
        if (red)
            fvb_check(plan.k.reduce(&plan.k, 0, n, args.data(), red, s));
        else
            fvb_check(plan.k.fn(&plan.k, 0, n, args.data(), s));
        // a reduction is read back (and waited for) by its caller, read_max
        if (be.synchronize && !red) cuda_check(cudaStreamSynchronize(s), "sync");
        return;
    }
    bool all_host = true;
    for (uint8_t d : on_dev) all_host = all_host && d != 1;
    double lam = 0.0;
    if (be.ordinals.size() > 1 && all_host) {
        lam = run_sliced(be, plan, n, args, prec, on_dev, red != nullptr, pass);
    } else {
        HostCtx& hc = host_ctx(be.ordinal);
        std::lock_guard<std::mutex> lock(hc.mu);
        if (!hc.ctx) fvb_check(fvb_ctx_create(be.ordinal, be.chunk_points, &hc.ctx));
        fvb_status st;
        {
            HostCopies copies(pass);  // joined before the result is returned
            st = fvb_launch_host(hc.ctx, &plan.k, n, args.data(), prec.data(), on_dev.data(),
                                 red ? &lam : nullptr, be.stream);
        }
        fvb_check(st);
    }
    if (red) {  // hand the maximum back through the caller's device scalar, in stream order
        const float f = static_cast<float>(lam);
        cuda_check(cudaMemcpyAsync(red, plan.k.prec ? static_cast<const void*>(&lam) : &f,
                                   plan.k.prec ? sizeof lam : sizeof f, cudaMemcpyHostToDevice, s),
                   "lambda");
        cuda_check(cudaStreamSynchronize(s), "lambda");
    }
}

// Look up the fused kernel for `items` writing `outs`; single items use the
// reference's expression key, several the block key.
bool try_plan(const std::vector<Expr>& items, std::vector<Out> outs, std::size_t rows,
              std::size_t cols, Plan* plan) {
    std::vector<Precision> dests;
    for (const Out& o : outs) dests.push_back(o.prec());
    std::vector<const DenseVector*> leaves;
    std::string key;
    if (items.size() == 1) {
        Slots slots;
        bool ok = true;
        key.assign(1, prec_char(dests[0]));
        key_node(items[0].node(), slots, ok, key);
        if (!ok) return false;
        leaves = slots.v;
    } else {
        key = block_key(items, dests, rows, cols, &leaves);
        if (key.empty()) return false;
    }
    fvb_kernel k;
    // Only "no kernel for this key" is a miss; a device or host failure while
    // lowering (NVRTC, module load) surfaces as its own exception.
    const fvb_status st = fvb_lookup(key.c_str(), &k);
    if (st == FVB_EUNSUPPORTED) return false;
    fvb_check(st);
    if (k.n_outputs != outs.size() || k.n_inputs != leaves.size()) return false;
    plan->k = k;
    plan->leaves = std::move(leaves);
    plan->outs = std::move(outs);
    return true;
}

[[noreturn]] void unsupported(const std::vector<Expr>& items) {
    std::string k = items.size() == 1 ? structural_key(items[0], items[0].result_precision())
                                      : std::string("block of ") + std::to_string(items.size()) +
                                            " items";
    throw UnsupportedExpression("no fused device kernel for " + k.substr(0, 200) +
                                " (general lowering is not implemented; no CPU fallback)");
}

// A device allocation freed on scope exit.
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(std::size_t bytes) {
        if (bytes) cuda_check(cudaMalloc(&p, bytes), "device allocation");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// CSR block-matvec rows (proj/src/block.cpp:389-411, 429-447): each row item
// y = sum_t M_t * eval(op_t) in the destination's precision.  Operands are
// device planes: a bare leaf is used in place when resident (else uploaded
// once), any other operand expression is evaluated once on the device into
// a scratch plane -- the reference's "one scratch per distinct operand".
// As in the reference, every operand is captured before any destination is
// written (a snapshot: y = M * y swaps correctly), and a resident operand
// whose plane is itself a destination is copied first, not used in place.
struct MatvecOperands {
    std::map<const ExprNode*, std::unique_ptr<DeviceVector>> owned;
    std::map<const ExprNode*, const DeviceVector*> planes;
    const DeviceVector& at(const Expr& op) const { return *planes.at(op.ptr().get()); }
};

// Every operand of the block's matvec rows, captured before any of the
// block's destinations (`dests`: all of them, element-wise items' included)
// is written.
void capture_operands(const DeviceBackend& be,
                      const std::vector<std::pair<const BlockItem*, Out>>& mv,
                      const std::vector<Out>& dests, MatvecOperands& ops) {
    DeviceGuard guard(be.ordinal);
    cudaStream_t s = static_cast<cudaStream_t>(be.stream);
    auto& owned = ops.owned;
    auto& planes = ops.planes;
    auto is_dest_plane = [&](const DeviceVector* p) {
        for (const Out& o : dests)
            if (o.dev == p) return true;
        return false;
    };
    auto capture = [&](const Expr& op, std::size_t cols) {
        const ExprNode* key = op.ptr().get();
        if (planes.count(key)) return;
        if (const DenseVector* lf = bare_leaf(op.node())) {
            if (lf->size() != cols)
                throw LengthMismatch("matvec column count " + std::to_string(cols) +
                                     " vs operand length " + std::to_string(lf->size()));
            DeviceVector* dv = be.residency ? be.residency->find(lf) : nullptr;
            if (dv && !is_dest_plane(dv)) {
                planes[key] = dv;
                return;
            }
            auto t = std::make_unique<DeviceVector>(lf->precision(), lf->size());
            if (dv) {  // the resident plane is written by this block: a snapshot
                if (dv->size() != lf->size() || dv->precision() != lf->precision())
                    throw LengthMismatch("resident plane does not match its host leaf");
                if (t->byte_size())
                    cuda_check(cudaMemcpyAsync(t->data(), dv->data(), t->byte_size(),
                                               cudaMemcpyDeviceToDevice, s),
                               "matvec operand snapshot");
            } else {
                t->upload(*lf);
            }
            planes[key] = t.get();
            owned[key] = std::move(t);
            return;
        }
        auto t = std::make_unique<DeviceVector>(op.result_precision(), cols);
        evaluate(be, op, *t);
        planes[key] = t.get();
        owned[key] = std::move(t);
    };
    for (const auto& [item, d] : mv)
        for (const MatVecTerm& t : item->terms()) capture(t.operand, t.mat->cols());
}

// One matvec row item into its destination, from captured operands.
void run_matvec_item(const DeviceBackend& be, const BlockItem* item, const Out& d,
                     const MatvecOperands& ops) {
    DeviceGuard guard(be.ordinal);
    cudaStream_t s = static_cast<cudaStream_t>(be.stream);
    const std::size_t rows = d.size();
    std::unique_ptr<DeviceVector> tmp;
    DeviceVector* y = d.dev;
    if (!y) {
        tmp = std::make_unique<DeviceVector>(d.prec(), rows);
        y = tmp.get();
    }
    if (rows) cuda_check(cudaMemsetAsync(y->data(), 0, y->byte_size(), s), "matvec reset");
    for (const MatVecTerm& t : item->terms()) {
        if (t.mat->rows() != rows)
            throw LengthMismatch("matvec row count " + std::to_string(t.mat->rows()) +
                                 " vs destination length " + std::to_string(rows));
        const DeviceVector& x = ops.at(t.operand);
        if (x.size() != t.mat->cols())
            throw LengthMismatch("matvec column count " + std::to_string(t.mat->cols()) +
                                 " vs operand length " + std::to_string(x.size()));
        const int py = y->precision() == Precision::f64 ? 1 : 0;
        const int px = x.precision() == Precision::f64 ? 1 : 0;
        if (const DeviceCsr* dm = be.residency ? be.residency->find(t.mat) : nullptr) {
            // a resident matrix: no upload
            if (dm->narrow_indices())
                fvb_check(fvb_csr_matvec_acc_u32(py, px, rows, dm->nnz(), dm->row_ptr(),
                                                 dm->col_idx32(), dm->values(), x.data(),
                                                 y->data(), s));
            else
                fvb_check(fvb_csr_matvec_acc(py, px, rows, dm->nnz(), dm->row_ptr(),
                                             dm->col_idx(), dm->values(), x.data(), y->data(),
                                             s));
            continue;
        }
        const auto& rp = t.mat->row_ptr();
        const auto& ci = t.mat->col_idx();
        const auto& v = t.mat->values();
        static_assert(sizeof(std::size_t) == sizeof(uint64_t), "64-bit size_t");
        DevBuf drp(rp.size() * 8), dci(ci.size() * 8), dv(v.size() * 8);
        if (!rp.empty())
            cuda_check(cudaMemcpyAsync(drp.p, rp.data(), rp.size() * 8, cudaMemcpyHostToDevice, s), "csr upload");
        if (!ci.empty()) {
            cuda_check(cudaMemcpyAsync(dci.p, ci.data(), ci.size() * 8, cudaMemcpyHostToDevice, s), "csr upload");
            cuda_check(cudaMemcpyAsync(dv.p, v.data(), v.size() * 8, cudaMemcpyHostToDevice, s), "csr upload");
        }
        fvb_check(fvb_csr_matvec_acc(py, px, rows, ci.size(),
                                     static_cast<const uint64_t*>(drp.p),
                                     static_cast<const uint64_t*>(dci.p),
                                     static_cast<const double*>(dv.p), x.data(), y->data(), s));
        cuda_check(cudaStreamSynchronize(s), "matvec");  // before the CSR buffers go
    }
    cuda_check(cudaStreamSynchronize(s), "matvec");
    if (d.host && rows)
        cuda_check(cudaMemcpy(d.host->raw(), y->data(), y->byte_size(), cudaMemcpyDeviceToHost),
                   "matvec read-back");
}

// CSR block-matvec rows of a block, operands captured first.
void run_matvec(const DeviceBackend& be, std::vector<std::pair<const BlockItem*, Out>>& mv,
                const std::vector<Out>& dests) {
    MatvecOperands ops;
    capture_operands(be, mv, dests, ops);
    for (const auto& [item, d] : mv) run_matvec_item(be, item, d, ops);
}

void leaves_of(const ExprNode& n, std::vector<const DenseVector*>& out) {
    switch (n.kind) {
        case NodeKind::Leaf: out.push_back(n.vec); return;
        case NodeKind::Constant: return;
        case NodeKind::Tagged:
        case NodeKind::Cached:
        case NodeKind::Unary: leaves_of(*n.left, out); return;
        case NodeKind::Binary:
            leaves_of(*n.left, out);
            leaves_of(*n.right, out);
            return;
    }
}

// True when some element-wise item reads a vector that an earlier item of
// the block writes (or that a matvec row writes: those run first here).
bool reads_earlier_destination(const DeviceBackend& be, const std::vector<Expr>& items,
                               const std::vector<Out>& outs,
                               const std::vector<std::pair<const BlockItem*, Out>>& matvecs) {
    // The earliest item writing each destination (a host vector, or a device
    // plane that is some leaf's resident copy); matvec rows count as written
    // before every item.  Linear in the leaves, so a 75-item Jacobian block
    // costs one pass over its trees.
    // (address, earliest writing item) sorted by address: a block has at most
    // a few hundred destinations, so a binary search beats hashing here
    std::vector<std::pair<const void*, long>> writer;
    writer.reserve(matvecs.size() + outs.size());
    for (const auto& mv : matvecs) {
        const Out& o = mv.second;
        if (o.host || o.dev) writer.push_back({o.host ? static_cast<const void*>(o.host) : o.dev, -1});
    }
    for (std::size_t j = 0; j < outs.size(); ++j) {
        const Out& o = outs[j];
        if (o.host || o.dev)
            writer.push_back({o.host ? static_cast<const void*>(o.host) : o.dev, long(j)});
    }
    if (writer.empty()) return false;
    std::sort(writer.begin(), writer.end());  // equal addresses: the earliest writer first
    auto earliest = [&](const void* p) -> long {
        auto it = std::lower_bound(writer.begin(), writer.end(), std::make_pair(p, long(-2)));
        return it != writer.end() && it->first == p ? it->second : long(items.size());
    };
    std::vector<const DenseVector*> ls;
    for (std::size_t k = 0; k < items.size(); ++k) {
        ls.clear();
        leaves_of(items[k].node(), ls);
        for (const DenseVector* l : ls) {
            if (earliest(l) < long(k)) return true;
            if (const DeviceVector* dv = be.residency ? be.residency->find(l) : nullptr)
                if (earliest(dv) < long(k)) return true;
        }
    }
    return false;
}

// A block with more planes than one launch's argument block carries runs as
// several fused kernels over halves of its items.  No item reads another's
// destination (block_impl checks that first), so the split is exact.  A
// single item that still has no kernel is unsupported.
void run_in_parts(const DeviceBackend& be, const std::vector<Expr>& items,
                  const std::vector<Out>& outs, std::size_t n) {
    Plan p;
    if (try_plan(items, outs, items.size(), 1, &p)) {
        run(be, p, n, nullptr);
        return;
    }
    if (items.size() == 1) unsupported(items);
    const std::size_t h = items.size() / 2;
    run_in_parts(be, std::vector<Expr>(items.begin(), items.begin() + long(h)),
                 std::vector<Out>(outs.begin(), outs.begin() + long(h)), n);
    run_in_parts(be, std::vector<Expr>(items.begin() + long(h), items.end()),
                 std::vector<Out>(outs.begin() + long(h), outs.end()), n);
}

// ---- the launch-plan cache of block evaluations ------------------------------
//
// A time loop evaluates the same BlockExpr object into the same destinations
// step after step: the expression objects are built once, and their leaves
// refer to the state vectors, which are updated in place.  Everything
// block_impl decides before the launch -- validating the trees, the aliasing
// analysis, the structural key, the kernel lookup, the host-side writes --
// is a function of the items' tree nodes (immutable), of the destinations'
// and leaves' identities and of the residency mapping.  Only the lengths and
// precisions of the vectors can change between calls (DenseVector and
// DeviceVector assignment).  So the decision is cached per thread, keyed by
// node and vector identities plus the Residency's version; each entry holds
// its item trees alive, so no cached address can come back as another tree.
// Lengths and precisions are checked again on every hit; any change misses,
// and the full path validates (and reports) it.  The reference re-derives
// its JIT key on every call (backend_jit.cpp:314-335); this is the device
// path's zero-overhead answer for reused expressions (profiles/r02_devbench_*).
struct BlockEntry {
    std::vector<const void*> ids;  // per item: root ExprNode, or a Vector item's DenseVector
    std::vector<std::shared_ptr<const ExprNode>> hold;
    std::vector<Out> dests;
    std::size_t rows = 0, cols = 0;
    bool reduce = false;
    const Residency* res = nullptr;
    std::uint64_t res_version = 0;
    // the decision
    Plan plan;
    std::vector<std::pair<const DenseVector*, Out>> copies;
    std::size_t n = 0;
    std::vector<Precision> dest_prec;
    std::vector<std::pair<const DenseVector*, Precision>> reads;  // every leaf read
};

constexpr std::size_t kBlockCacheEntries = 8;

std::vector<std::unique_ptr<BlockEntry>>& block_cache() {
    thread_local std::vector<std::unique_ptr<BlockEntry>> c;
    return c;
}

bool same_out(const Out& a, const Out& b) {
    return a.host == b.host && a.dev == b.dev && a.null_prec == b.null_prec &&
           a.null_size == b.null_size;
}

// The identities of e's items; false when some item cannot be cached (a
// matvec row or a matrix item: those paths upload and allocate per call).
bool item_ids(const BlockExpr& e, std::size_t rows, std::size_t cols,
              std::vector<const void*>& ids) {
    ids.clear();
    for (std::size_t r = 0; r < rows; ++r)
        for (std::size_t c = 0; c < cols; ++c) {
            const BlockItem& it = e.item(r, c);
            if (it.kind() == ItemKind::Expression && it.expr().valid())
                ids.push_back(it.expr().ptr().get());
            else if (it.kind() == ItemKind::Vector)
                ids.push_back(&it.vector());
            else
                return false;
        }
    return true;
}

BlockEntry* cached_block(const DeviceBackend& be, const std::vector<const void*>& ids,
                         std::size_t rows, std::size_t cols, const std::vector<Out>& dests,
                         bool reduce) {
    auto& cache = block_cache();
    for (std::size_t i = 0; i < cache.size(); ++i) {
        BlockEntry& c = *cache[i];
        if (c.rows != rows || c.cols != cols || c.reduce != reduce || c.res != be.residency ||
            (be.residency && c.res_version != be.residency->version()) || c.ids != ids ||
            c.dests.size() != dests.size())
            continue;
        bool same = true;
        for (std::size_t j = 0; j < dests.size() && same; ++j) same = same_out(c.dests[j], dests[j]);
        if (!same) continue;
        // lengths and precisions as when the decision was made
        for (std::size_t j = 0; j < dests.size() && same; ++j)
            same = dests[j].size() == c.n && dests[j].prec() == c.dest_prec[j];
        for (const auto& [v, p] : c.reads) same = same && v->size() == c.n && v->precision() == p;
        if (!same) return nullptr;
        if (i) std::rotate(cache.begin(), cache.begin() + long(i), cache.begin() + long(i) + 1);
        return cache.front().get();
    }
    return nullptr;
}

void remember_block(const DeviceBackend& be, const BlockExpr& e, std::vector<const void*> ids,
                    std::size_t rows, std::size_t cols, const std::vector<Out>& dests, bool reduce,
                    const Plan& plan,
                    const std::vector<std::pair<const DenseVector*, Out>>& copies,
                    std::size_t n) {
    auto ent = std::make_unique<BlockEntry>();
    ent->ids = std::move(ids);
    for (std::size_t r = 0; r < rows; ++r)
        for (std::size_t c = 0; c < cols; ++c) {
            const BlockItem& it = e.item(r, c);
            if (it.kind() == ItemKind::Expression) ent->hold.push_back(it.expr().ptr());
        }
    ent->dests = dests;
    ent->rows = rows;
    ent->cols = cols;
    ent->reduce = reduce;
    ent->res = be.residency;
    ent->res_version = be.residency ? be.residency->version() : 0;
    ent->plan = plan;
    ent->copies = copies;
    ent->n = n;
    for (const Out& d : dests) ent->dest_prec.push_back(d.prec());
    for (const DenseVector* l : plan.leaves) ent->reads.push_back({l, l->precision()});
    for (const auto& cp : copies) ent->reads.push_back({cp.first, cp.first->precision()});
    auto& cache = block_cache();
    if (cache.size() == kBlockCacheEntries) cache.pop_back();
    cache.insert(cache.begin(), std::move(ent));
}

// The launch and the pass-through copies of a decided block.
void run_block(const DeviceBackend& be, Plan& plan,
               const std::vector<std::pair<const DenseVector*, Out>>& copies, std::size_t n,
               void* red);

// Shared body of the evaluate_block overloads.
void block_impl(const DeviceBackend& be, const BlockExpr& e, std::size_t rows, std::size_t cols,
                const std::vector<Out>& dests_in, void* red, bool need_reduce) {
    if (e.block_rows() != rows || e.block_cols() != cols)
        throw ShapeMismatch("block expression shape " + std::to_string(e.block_rows()) + "x" +
                            std::to_string(e.block_cols()) + " does not match destination " +
                            std::to_string(rows) + "x" + std::to_string(cols));
    std::vector<const void*> ids;
    const bool cacheable = item_ids(e, rows, cols, ids);
    if (cacheable)
        if (BlockEntry* hit = cached_block(be, ids, rows, cols, dests_in, need_reduce)) {
            run_block(be, hit->plan, hit->copies, hit->n, red);
            return;
        }
    const std::size_t rows_in = rows, cols_in = cols;
    std::vector<Expr> items;
    std::vector<Out> outs;
    std::vector<std::pair<const DenseVector*, Out>> copies;  // bare-leaf items
    std::vector<std::pair<const BlockItem*, Out>> matvecs;   // CSR block-matvec rows
    std::vector<std::pair<bool, std::size_t>> order;  // (matvec?, index): the reference's item order
    std::size_t idx = 0;
    for (std::size_t r = 0; r < rows; ++r)
        for (std::size_t c = 0; c < cols; ++c, ++idx) {
            const BlockItem& it = e.item(r, c);
            Expr x;
            switch (it.kind()) {
                case ItemKind::Expression: x = it.expr(); break;
                case ItemKind::Vector: x = leaf(it.vector()); break;
                case ItemKind::MatVec:
                    if (need_reduce) throw UnsupportedExpression("matvec block has no CFL reduction");
                    order.push_back({true, matvecs.size()});
                    matvecs.push_back({&it, dests_in[idx]});
                    continue;
                default:  // as the reference: proj/src/block.cpp:427-428
                    throw KindMismatch("cannot assign a sparse-matrix item into a vector");
            }
            const Out& d = dests_in[idx];
            std::map<int, const DenseVector*> tags;
            validate(x.node(), d.size(), tags);
            // aliased pass-through moves no memory (proj/src/block.cpp:419-422)
            if (d.host && bare_leaf(x.node()) == d.host) continue;
            order.push_back({false, items.size()});
            items.push_back(x);
            outs.push_back(d);
        }
    // The reference writes items one by one (block.cpp:413-451), so an item
    // reading a vector an earlier item of the same block wrote sees the new
    // values; one fused pass reads every operand before writing anything.
    // Such blocks are evaluated item by item instead, in the reference's order.
    bool hazard = reads_earlier_destination(be, items, outs, matvecs);
    // Two items writing one destination: the later one's value stands, as
    // item-by-item evaluation leaves it (the host-buffer pipeline refuses
    // one plane named for two outputs).
    // (Matvec rows count too: with them the order decides which value stands.)
    if (!hazard && !need_reduce) {
        std::vector<const void*> seen;
        seen.reserve(outs.size() + matvecs.size());
        auto note = [&](const Out& o) {
            if (o.host || o.dev) seen.push_back(o.host ? static_cast<const void*>(o.host) : o.dev);
        };
        for (const Out& o : outs) note(o);
        for (const auto& m : matvecs) note(m.second);
        std::sort(seen.begin(), seen.end());
        hazard = std::adjacent_find(seen.begin(), seen.end()) != seen.end();
    }
    if (hazard && need_reduce)
        throw UnsupportedExpression(
            "CFL block whose destinations alias operands of its own items");
    if (hazard) {
        // The reference's own order (block.cpp:389-451): every matvec operand
        // captured first, then the items one by one, so an item reading an
        // earlier item's destination sees the new values and a later one's
        // the old.
        MatvecOperands ops;
        if (!matvecs.empty()) capture_operands(be, matvecs, dests_in, ops);
        for (const auto& [is_mv, k] : order) {
            if (is_mv) {
                run_matvec_item(be, matvecs[k].first, matvecs[k].second, ops);
                continue;
            }
            Plan one;
            if (!try_plan({items[k]}, {outs[k]}, 1, 1, &one)) unsupported({items[k]});
            run(be, one, outs[k].size(), nullptr);
        }
        return;
    }
    // Matvec rows first: no element-wise item reads their destinations (no
    // hazard), and their operands are captured before any destination of this
    // block is written (the reference's scratch pass, block.cpp:389-411).
    if (!matvecs.empty()) run_matvec(be, matvecs, dests_in);
    if (items.empty()) return;
    const std::size_t n = outs[0].size();
    for (const Out& o : outs)
        if (o.size() != n) throw LengthMismatch("block destinations have different lengths");
    // Matvec rows or aliased pass-throughs were taken out: the fused key
    // covers the remaining element-wise items as one column.
    if (items.size() != rows * cols) {
        rows = items.size();
        cols = 1;
    }
    // Prefer a hand-written fused kernel: the whole block, else the block
    // without its bare-leaf items (plain copies, e.g. the density that
    // convert() passes through).  Only if neither exists, lower the whole
    // block (fvb_lookup's NVRTC path, plan.k.impl != NULL).
    Plan plan;
    const bool whole = try_plan(items, outs, rows, cols, &plan);
    if (!whole || plan.k.impl) {
        std::vector<Expr> rest;
        std::vector<Out> rest_outs;
        std::vector<std::pair<const DenseVector*, Out>> stripped;
        for (std::size_t i = 0; i < items.size(); ++i) {
            if (const DenseVector* src = bare_leaf(items[i].node()))
                stripped.push_back({src, outs[i]});
            else {
                rest.push_back(items[i]);
                rest_outs.push_back(outs[i]);
            }
        }
        // The stripped copies run after the kernel.  The reference copies
        // each one at its own position (block.cpp:413-451), so a later item
        // that overwrites a copy's source -- e.g. convert(u, Primitive) with
        // the pressure written over rho -- must not run first: such blocks
        // keep the bare-leaf items inside the fused pass, which reads every
        // leaf before it writes.  So must blocks where a computed item and a
        // copy name one destination.
        auto overwrites_a_source = [&] {
            for (const auto& [src, o] : stripped) {
                const DeviceVector* rs = be.residency ? be.residency->find(src) : nullptr;
                for (const Out& r : rest_outs) {
                    if ((r.host && r.host == src) || (r.dev && rs && r.dev == rs)) return true;
                    // one destination for both: the later item's value wins
                    if ((r.host && r.host == o.host) || (r.dev && r.dev == o.dev)) return true;
                }
            }
            return false;
        };
        Plan alt;
        if (!stripped.empty() && !rest.empty() && !overwrites_a_source() &&
            try_plan(rest, rest_outs, rest.size(), 1, &alt) && (!alt.k.impl || !whole)) {
            plan = std::move(alt);
            copies = std::move(stripped);
        } else if (!whole) {
            if (need_reduce) unsupported(items);
            run_in_parts(be, items, outs, n);
            return;
        }
    }
    if (need_reduce && !plan.k.reduce)
        throw UnsupportedExpression("block has no fused CFL reduction");
    if (copies.empty() && plan.outs.size() == items.size()) {
        // bare-leaf items of a fused block whose source and destination are
        // both host vectors of one precision, and whose source no item
        // overwrites: copied host-side while the device pipeline runs
        // ... and bare constant items of host destinations are filled
        // host-side (the Jacobian's 30 constant entries of 75 in 3-D)
        plan.pass_src.assign(plan.outs.size(), nullptr);
        plan.has_fill.assign(plan.outs.size(), 0);
        plan.fill_bits.assign(plan.outs.size(), 0);
        // Host-side writes run concurrently with the device pipeline, so
        // their destination must be no leaf of the block (the kernel may
        // still be reading it) and no other item's destination.
        auto exclusive = [&](const DenseVector* d) {
            for (const DenseVector* l : plan.leaves)
                if (l == d) return false;
            std::size_t uses = 0;
            for (const Out& w : plan.outs) uses += w.host == d;
            return uses == 1;
        };
        // (The hand-written Jacobian's constant and duplicate entries are
        // written host-side by fvb_launch_host itself, with streaming stores.)
        const bool lib_fills = !plan.k.impl && std::strncmp(plan.k.name, "jacobian", 8) == 0;
        for (std::size_t j = 0; j < items.size(); ++j) {
            const Out& o = plan.outs[j];
            if (!o.host || !exclusive(o.host)) continue;
            if (!lib_fills &&
                bare_constant(items[j].node(), o.host->precision(), &plan.fill_bits[j])) {
                plan.has_fill[j] = 1;
                continue;
            }
            const DenseVector* src = bare_leaf(items[j].node());
            if (!src || !o.host || o.host->precision() != src->precision() ||
                (be.residency && be.residency->find(src)))
                continue;
            bool written = false;
            for (const Out& w : plan.outs) written |= w.host == src;
            if (!written) plan.pass_src[j] = src;
        }
    }
    if (cacheable)
        remember_block(be, e, std::move(ids), rows_in, cols_in, dests_in, need_reduce, plan, copies,
                       n);
    run_block(be, plan, copies, n, red);
}

void run_block(const DeviceBackend& be, Plan& plan,
               const std::vector<std::pair<const DenseVector*, Out>>& copies, std::size_t n,
               void* red) {
    run(be, plan, n, red);
    // Pass-through items: plain copies.  A device destination is filled in
    // stream order on the backend's stream -- from the leaf's resident plane
    // when it has one -- so asynchronous (and graph-captured) evaluations
    // stay asynchronous.
    cudaStream_t s = static_cast<cudaStream_t>(be.stream);
    bool queued = false;
    for (const auto& [src, d] : copies) {
        DeviceGuard guard(be.ordinal);
        if (d.host) {
            std::memcpy(d.host->raw(), src->raw(), d.host->byte_size());
            continue;
        }
        const DeviceVector* rs = be.residency ? be.residency->find(src) : nullptr;
        cuda_check(cudaMemcpyAsync(d.dev->data(), rs ? rs->data() : src->raw(), d.dev->byte_size(),
                                   rs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s),
                   "pass-through copy");
        queued = true;
    }
    if (queued && be.synchronize) cuda_check(cudaStreamSynchronize(s), "pass-through copy");
}

// The maximum a reduction left in the device word, read back in stream
// order on the backend's stream through a pinned word: one wait for the
// kernel and the copy together.
double read_max(const DeviceBackend& be, void* red, Precision p) {
    struct Pinned {
        void* p = nullptr;
        ~Pinned() {
            if (p) cudaFreeHost(p);
        }
    };
    thread_local Pinned host;
    if (!host.p) cuda_check(cudaHostAlloc(&host.p, 8, cudaHostAllocDefault), "pinned word");
    cudaStream_t s = static_cast<cudaStream_t>(be.stream);
    DeviceGuard guard(be.ordinal);
    cuda_check(cudaMemcpyAsync(host.p, red, p == Precision::f64 ? 8 : 4, cudaMemcpyDeviceToHost, s),
               "lambda read-back");
    cuda_check(cudaStreamSynchronize(s), "lambda read-back");
    if (p == Precision::f64) return *static_cast<const double*>(host.p);
    return double(*static_cast<const float*>(host.p));
}

// The CFL accumulator: one 8-byte device word per host thread and device
// (reused across calls), zeroed in stream order on the backend's stream
// before each reduction.
struct DeviceScalar {
    void* p = nullptr;
    explicit DeviceScalar(const DeviceBackend& be) {
        struct Cache {
            std::map<int, void*> words;
            ~Cache() {
                for (auto& w : words) cudaFree(w.second);
            }
        };
        thread_local Cache cache;
        DeviceGuard guard(be.ordinal);
        void*& word = cache.words[be.ordinal];
        if (!word) cuda_check(cudaMalloc(&word, 8), "scalar allocation");
        p = word;
        cuda_check(cudaMemsetAsync(p, 0, 8, static_cast<cudaStream_t>(be.stream)), "scalar reset");
    }
};

}  // namespace

// ---- DeviceVector / Residency ------------------------------------------------

DeviceVector::DeviceVector(Precision prec, std::size_t len) : prec_(prec), len_(len) {
    if (len_) cuda_check(cudaMalloc(&ptr_, byte_size()), "DeviceVector allocation");
}

DeviceVector::~DeviceVector() {
    if (ptr_) cudaFree(ptr_);
}

DeviceVector::DeviceVector(DeviceVector&& o) noexcept : prec_(o.prec_), len_(o.len_), ptr_(o.ptr_) {
    o.ptr_ = nullptr;
    o.len_ = 0;
}

DeviceVector& DeviceVector::operator=(DeviceVector&& o) noexcept {
    if (this != &o) {
        if (ptr_) cudaFree(ptr_);
        prec_ = o.prec_;
        len_ = o.len_;
        ptr_ = o.ptr_;
        o.ptr_ = nullptr;
        o.len_ = 0;
    }
    return *this;
}

void DeviceVector::upload(const DenseVector& host) {
    if (host.size() != len_) throw LengthMismatch("upload: length differs");
    if (host.precision() != prec_) throw Error("upload: precision differs");
    if (len_) cuda_check(cudaMemcpy(ptr_, host.raw(), byte_size(), cudaMemcpyHostToDevice), "upload");
}

void DeviceVector::download(DenseVector& host) const {
    if (host.size() != len_) throw LengthMismatch("download: length differs");
    if (host.precision() != prec_) throw Error("download: precision differs");
    if (len_)
        cuda_check(cudaMemcpy(host.raw(), ptr_, byte_size(), cudaMemcpyDeviceToHost), "download");
}

DeviceVector make_temp(Precision prec, std::size_t len) { return DeviceVector(prec, len); }

namespace {
std::uint64_t fresh_version() {
    static std::atomic<std::uint64_t> next{1};
    return next.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace

Residency::Residency() : version_(fresh_version()) {}

Residency::Residency(const Residency& o) : map_(o.map_), csr_(o.csr_), version_(fresh_version()) {}

Residency& Residency::operator=(const Residency& o) {
    if (this != &o) {
        map_ = o.map_;
        csr_ = o.csr_;
        version_ = fresh_version();
    }
    return *this;
}

void Residency::bind(const DenseVector& host, DeviceVector& dev) {
    if (host.size() != dev.size()) throw LengthMismatch("bind: length differs");
    map_[&host] = &dev;
    version_ = fresh_version();
}

void Residency::unbind(const DenseVector& host) {
    map_.erase(&host);
    version_ = fresh_version();
}

DeviceVector* Residency::find(const DenseVector* host) const {
    auto it = map_.find(host);
    return it == map_.end() ? nullptr : it->second;
}

void Residency::bind(const SparseMatrix& host, DeviceCsr& dev) {
    if (host.rows() != dev.rows() || host.cols() != dev.cols() || host.nnz() != dev.nnz())
        throw ShapeMismatch("bind: the device CSR copy has another shape");
    csr_[&host] = &dev;
    version_ = fresh_version();
}

void Residency::unbind(const SparseMatrix& host) {
    csr_.erase(&host);
    version_ = fresh_version();
}

DeviceCsr* Residency::find(const SparseMatrix* host) const {
    auto it = csr_.find(host);
    return it == csr_.end() ? nullptr : it->second;
}

DeviceCsr::DeviceCsr(const SparseMatrix& m, int ordinal) : ordinal_(ordinal) { upload(m); }

DeviceCsr::~DeviceCsr() {
    if (rp_) cudaFree(rp_);
    if (ci_) cudaFree(ci_);
    if (v_) cudaFree(v_);
}

void DeviceCsr::upload(const SparseMatrix& m) {
    static_assert(sizeof(std::size_t) == sizeof(std::uint64_t), "64-bit size_t");
    DeviceGuard guard(ordinal_);
    const bool narrow = m.cols() <= std::size_t(UINT32_MAX);
    if (m.rows() != rows_ || m.nnz() != nnz_ || narrow != narrow_ || !rp_) {
        if (rp_) cudaFree(rp_);
        if (ci_) cudaFree(ci_);
        if (v_) cudaFree(v_);
        rp_ = nullptr;
        ci_ = nullptr;
        v_ = nullptr;
        cuda_check(cudaMalloc(&rp_, (m.rows() + 1) * 8), "csr allocation");
        if (m.nnz()) {
            cuda_check(cudaMalloc(&ci_, m.nnz() * (narrow ? 4 : 8)), "csr allocation");
            cuda_check(cudaMalloc(&v_, m.nnz() * 8), "csr allocation");
        }
    }
    rows_ = m.rows();
    cols_ = m.cols();
    nnz_ = m.nnz();
    narrow_ = narrow;
    cuda_check(cudaMemcpy(rp_, m.row_ptr().data(), (rows_ + 1) * 8, cudaMemcpyHostToDevice),
               "csr upload");
    if (nnz_ && narrow_) {
        // the once-per-upload narrowing: every index < cols <= 2^32 - 1
        const std::vector<std::size_t>& ci = m.col_idx();
        std::vector<std::uint32_t> ci32(ci.begin(), ci.end());
        cuda_check(cudaMemcpy(ci_, ci32.data(), nnz_ * 4, cudaMemcpyHostToDevice), "csr upload");
        cuda_check(cudaMemcpy(v_, m.values().data(), nnz_ * 8, cudaMemcpyHostToDevice),
                   "csr upload");
    } else if (nnz_) {
        cuda_check(cudaMemcpy(ci_, m.col_idx().data(), nnz_ * 8, cudaMemcpyHostToDevice),
                   "csr upload");
        cuda_check(cudaMemcpy(v_, m.values().data(), nnz_ * 8, cudaMemcpyHostToDevice),
                   "csr upload");
    }
}

// ---- keys ---------------------------------------------------------------------

std::string structural_key(const Expr& e, Precision dest) {
    Slots slots;
    bool ok = true;
    std::string key(1, prec_char(dest));
    key_node(e.node(), slots, ok, key);
    return ok ? key : std::string();
}

std::string block_key(const std::vector<Expr>& items, const std::vector<Precision>& dests,
                      std::size_t rows, std::size_t cols,
                      std::vector<const DenseVector*>* leaves) {
    Slots slots;
    bool ok = true;
    std::string key = "G" + std::to_string(rows) + "x" + std::to_string(cols) + ":";
    KeyOut w(key);
    for (std::size_t i = 0; i < items.size(); ++i) {
        if (i) w.put('|');
        w.put(prec_char(dests[i]));
        key_node(items[i].node(), slots, ok, w);
    }
    w.finish();
    if (leaves) *leaves = slots.v;
    return ok ? key : std::string();
}

// ---- evaluation -----------------------------------------------------------------

namespace {

// The single-expression counterpart of the block launch-plan cache (see
// BlockEntry): keyed by the tree's root node, the destination's identity and
// the residency version; lengths and precisions checked on every hit.
struct ExprEntry {
    std::shared_ptr<const ExprNode> root;
    Out dest;
    const Residency* res = nullptr;
    std::uint64_t res_version = 0;
    Plan plan;
    std::size_t n = 0;
    Precision dest_prec = Precision::f64;
    std::vector<Precision> leaf_prec;
};

std::vector<std::unique_ptr<ExprEntry>>& expr_cache() {
    thread_local std::vector<std::unique_ptr<ExprEntry>> c;
    return c;
}

void evaluate_into(const DeviceBackend& be, const Expr& e, const Out& o) {
    if (!e.valid()) throw Error("cannot evaluate an empty expression");
    auto& cache = expr_cache();
    for (std::size_t i = 0; i < cache.size(); ++i) {
        ExprEntry& c = *cache[i];
        if (c.root.get() != e.ptr().get() || !same_out(c.dest, o) || c.res != be.residency ||
            (be.residency && c.res_version != be.residency->version()))
            continue;
        bool same = o.size() == c.n && o.prec() == c.dest_prec;
        for (std::size_t l = 0; l < c.plan.leaves.size() && same; ++l)
            same = c.plan.leaves[l]->size() == c.n && c.plan.leaves[l]->precision() == c.leaf_prec[l];
        if (!same) break;  // the full path validates (and reports) the change
        if (i) std::rotate(cache.begin(), cache.begin() + long(i), cache.begin() + long(i) + 1);
        run(be, cache.front()->plan, c.n, nullptr);
        return;
    }
    std::map<int, const DenseVector*> tags;
    validate(e.node(), o.size(), tags);
    if (o.size() == 0) return;
    auto ent = std::make_unique<ExprEntry>();
    if (!try_plan({e}, {o}, 1, 1, &ent->plan)) unsupported({e});
    ent->root = e.ptr();
    ent->dest = o;
    ent->res = be.residency;
    ent->res_version = be.residency ? be.residency->version() : 0;
    ent->n = o.size();
    ent->dest_prec = o.prec();
    for (const DenseVector* l : ent->plan.leaves) ent->leaf_prec.push_back(l->precision());
    if (cache.size() == kBlockCacheEntries) cache.pop_back();
    cache.insert(cache.begin(), std::move(ent));
    run(be, cache.front()->plan, o.size(), nullptr);
}

}  // namespace

void evaluate(const DeviceBackend& be, const Expr& e, DenseVector& dest) {
    Out o;
    o.host = &dest;
    evaluate_into(be, e, o);
}

void evaluate(const DeviceBackend& be, const Expr& e, DeviceVector& dest) {
    Out o;
    o.dev = &dest;
    evaluate_into(be, e, o);
}

void evaluate_block(const DeviceBackend& be, const BlockExpr& e, BlockVectorGrid& dest) {
    std::vector<Out> outs;
    for (std::size_t r = 0; r < dest.block_rows(); ++r)
        for (std::size_t c = 0; c < dest.block_cols(); ++c) {
            Out o;
            o.host = &dest.item(r, c);
            outs.push_back(o);
        }
    block_impl(be, e, dest.block_rows(), dest.block_cols(), outs, nullptr, false);
}

void evaluate_block(const DeviceBackend& be, const BlockExpr& e, BlockColVector& dest) {
    std::vector<Out> outs;
    for (std::size_t r = 0; r < dest.size(); ++r) {
        Out o;
        o.host = &dest.get(r);
        outs.push_back(o);
    }
    block_impl(be, e, dest.size(), 1, outs, nullptr, false);
}

void evaluate_block(const DeviceBackend& be, const BlockExpr& e, const Tie& dest) {
    if (dest.dests.size() != e.block_rows() * e.block_cols())
        throw ShapeMismatch("tie has " + std::to_string(dest.dests.size()) +
                            " destinations for a " + std::to_string(e.block_rows()) + "x" +
                            std::to_string(e.block_cols()) + " block");
    std::vector<Out> outs;
    for (DeviceVector* d : dest.dests) {
        Out o;
        o.dev = d;
        outs.push_back(o);
    }
    block_impl(be, e, e.block_rows(), e.block_cols(), outs, nullptr, false);
}

double reduce_max(const DeviceBackend& be, const Expr& lambda) {
    if (!lambda.valid()) throw Error("cannot reduce an empty expression");
    const Precision P = lambda.result_precision();
    Slots slots;
    bool ok = true;
    std::string key(1, prec_char(P));
    key_node(lambda.node(), slots, ok, key);
    Plan plan;
    if (!ok || fvb_lookup(key.c_str(), &plan.k) != FVB_OK || !plan.k.reduce)
        throw UnsupportedExpression("reduce_max needs a wave-speed expression (wave_speed(u))");
    plan.leaves = slots.v;
    const std::size_t n = plan.leaves.empty() ? 0 : plan.leaves[0]->size();
    std::map<int, const DenseVector*> tags;
    validate(lambda.node(), n, tags);
    Out none;  // NULL output slot: reduce only, no lambda plane
    none.null_prec = P;
    none.null_size = n;
    plan.outs = {none};
    DeviceScalar red(be);
    run(be, plan, n, red.p);
    return read_max(be, red.p, P);
}

double evaluate_block_cfl(const DeviceBackend& be, const BlockExpr& jacobian,
                          BlockVectorGrid& dest) {
    std::vector<Out> outs;
    for (std::size_t r = 0; r < dest.block_rows(); ++r)
        for (std::size_t c = 0; c < dest.block_cols(); ++c) {
            Out o;
            o.host = &dest.item(r, c);
            outs.push_back(o);
        }
    DeviceScalar red(be);
    block_impl(be, jacobian, dest.block_rows(), dest.block_cols(), outs, red.p, true);
    return read_max(be, red.p, dest.get(0).precision());
}

double evaluate_block_cfl(const DeviceBackend& be, const BlockExpr& jacobian, const Tie& dest) {
    std::vector<Out> outs;
    for (DeviceVector* d : dest.dests) {
        Out o;
        o.dev = d;
        outs.push_back(o);
    }
    DeviceScalar red(be);
    block_impl(be, jacobian, jacobian.block_rows(), jacobian.block_cols(), outs, red.p, true);
    return read_max(be, red.p, dest.dests.at(0)->precision());
}

void evaluate_block_cfl(const DeviceBackend& be, const BlockExpr& jacobian, const Tie& dest,
                        DeviceVector& lambda_max) {
    if (lambda_max.size() != 1 || dest.dests.empty() ||
        lambda_max.precision() != dest.dests.at(0)->precision())
        throw LengthMismatch("lambda_max must be one element of the block's precision");
    std::vector<Out> outs;
    for (DeviceVector* d : dest.dests) {
        Out o;
        o.dev = d;
        outs.push_back(o);
    }
    DeviceGuard guard(be.ordinal);
    cuda_check(cudaMemsetAsync(lambda_max.data(), 0, lambda_max.byte_size(),
                               static_cast<cudaStream_t>(be.stream)),
               "lambda reset");
    block_impl(be, jacobian, jacobian.block_rows(), jacobian.block_cols(), outs, lambda_max.data(),
               true);
    if (be.synchronize)
        cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(be.stream)), "sync");
}

}  // namespace device
}  // namespace fusevec
