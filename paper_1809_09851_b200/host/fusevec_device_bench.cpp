// fusevec_device_bench.cpp -- the reference's benchmark harness
// (proj/include/fusevec/bench.hpp, proj/src/bench.cpp) on the device backend.
//
// Same suites, same protocol, same records; only the two timed callables
// move to the device:
//
//   micro    y = (mx^2 + my^2 + mz^2) / rho^2    (bench.cpp:153-206)
//   miniapp  the full 5x3 inviscid flux block    (bench.cpp:294-384)
//
//   generic  the reference's own expression tree (derived_v_mag2(u),
//            inviscid_flux(u)) evaluated through the adapter's evaluate /
//            evaluate_block on every call: tree walk, validation, structural
//            key, kernel lookup, launch, completion -- what a user of the
//            reference's API pays;
//   hand     the fused kernel called directly through the C ABI, resolved
//            once outside the timed region (fvb_v_mag2 / fvb_flux on device
//            planes, fvb_launch_host / fvb_flux_host on host planes) -- the
//            device counterpart of the reference's hand-fused loops.
//
// overhead_ratio = median(generic) / median(hand) is then the paper's
// zero-overhead question asked of the device backend: what the generic
// expression API costs over a hand-written fused call.  Each callable returns
// only once its results are in place (the reference's time_ns wraps a
// synchronous call), interleaved ABAB, reps per decide_reps (>= 200 ms and
// >= 3), medians -- bench.cpp:46-51, 182-195, 360-371.
//
// Checks per size, outside the timed region, as the reference's harness does
// (OracleMismatch on failure): generic == hand bit for bit; generic == the
// reference's own Backend::scalar_ref() bit for bit (the device path's parity
// claim); miniapp also the element-wise flux oracle at the reference's sample
// points and tolerance (bench.cpp:321-336).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "fusevec_device.hpp"
#include "fvb.h"

namespace fusevec {
namespace device {

namespace {

using Clock = std::chrono::steady_clock;

template <class F>
double time_ns(F&& fn) {
    const auto t0 = Clock::now();
    fn();
    const auto t1 = Clock::now();
    return static_cast<double>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
}

double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const std::size_t m = v.size() / 2;
    return v.size() % 2 ? v[m] : 0.5 * (v[m - 1] + v[m]);
}

// bench.cpp:46-51
int decide_reps(const BenchConfig& cfg, double pair_ns) {
    if (cfg.reps > 0) return cfg.reps;
    const double want = 200e6;  // >= 200 ms per size
    const double r = std::ceil(want / std::max(pair_ns, 1.0));
    return static_cast<int>(std::clamp(r, 3.0, 2e6));
}

// The reference's smooth positive profile, same operations in the same
// order (bench.cpp:55-75): rho = 1 + 0.1 sin(2 pi i / n), v = (0.1, 0.2,
// 0.3), p = 1, rhoE from the perfect-gas closure; set() narrows for f32.
struct Profile {
    DenseVector rho, mx, my, mz, rho_E;
};

Profile make_profile(std::size_t n, Precision prec) {
    Profile f{DenseVector(prec, n), DenseVector(prec, n), DenseVector(prec, n),
              DenseVector(prec, n), DenseVector(prec, n)};
    const double vx = 0.1, vy = 0.2, vz = 0.3, p = 1.0;
    const double gm1 = 0.4;
    const double two_pi = 6.283185307179586;
    for (std::size_t i = 0; i < n; ++i) {
        const double rho =
            1.0 + 0.1 * std::sin(two_pi * static_cast<double>(i) / static_cast<double>(n));
        f.rho.set(i, rho);
        f.mx.set(i, rho * vx);
        f.my.set(i, rho * vy);
        f.mz.set(i, rho * vz);
        f.rho_E.set(i, p / gm1 + 0.5 * rho * (vx * vx + vy * vy + vz * vz));
    }
    return f;
}

bool same_bits(const DenseVector& a, const DenseVector& b) {
    return a.precision() == b.precision() && a.size() == b.size() &&
           std::memcmp(a.raw(), b.raw(), a.byte_size()) == 0;
}

void check_no_alloc(std::uint64_t before, const char* where) {
    if (vector_alloc_count() != before)
        throw Error(std::string("vector allocation inside the timed region of ") + where);
}

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw DeviceError(std::string(what) + ": " + cudaGetErrorName(e));
}

void fvb_ok(fvb_status st, const char* what) {
    if (st != FVB_OK) throw DeviceError(std::string(what) + ": " + fvb_last_error());
}

// bench.cpp:86-98: one flop per op node, reads = distinct leaves.
std::size_t count_ops(const ExprNode& n) {
    std::size_t c = (n.kind == NodeKind::Unary || n.kind == NodeKind::Binary) ? 1 : 0;
    if (n.left) c += count_ops(*n.left);
    if (n.right) c += count_ops(*n.right);
    return c;
}

void collect_leaves(const ExprNode& n, std::set<const DenseVector*>& out) {
    if (n.kind == NodeKind::Leaf) out.insert(n.vec);
    if (n.left) collect_leaves(*n.left, out);
    if (n.right) collect_leaves(*n.right, out);
}

// bench.cpp:261-272, in double
double flux_oracle(const Profile& f, std::size_t r, std::size_t c, std::size_t i) {
    const double rho = f.rho.at(i);
    const double m[3] = {f.mx.at(i), f.my.at(i), f.mz.at(i)};
    const double rho_E = f.rho_E.at(i);
    const double msq = m[0] * m[0] + m[1] * m[1] + m[2] * m[2];
    const double p = 0.4 * (rho_E - 0.5 * (msq / rho));
    const double v_c = m[c] / rho;
    if (r == 0) return m[c];
    if (r <= 3) return m[r - 1] * v_c + (r - 1 == c ? p : 0.0);
    return v_c * (rho_E + p);
}

// The device-resident copy of a profile, bound for the generic path.
struct Resident {
    std::vector<DeviceVector> planes;
    Residency res;
    explicit Resident(const Profile& f) {
        for (const DenseVector* v : {&f.rho, &f.mx, &f.my, &f.mz, &f.rho_E}) {
            planes.emplace_back(v->precision(), v->size());
            planes.back().upload(*v);
        }
        const DenseVector* hv[5] = {&f.rho, &f.mx, &f.my, &f.mz, &f.rho_E};
        for (int i = 0; i < 5; ++i) res.bind(*hv[i], planes[size_t(i)]);
    }
    std::vector<const void*> ptrs() const {
        std::vector<const void*> p;
        for (const auto& d : planes) p.push_back(d.data());
        return p;
    }
};

// An fvb_ctx for the hand path on host planes (fvb_*_host).
struct Ctx {
    fvb_ctx* c = nullptr;
    Ctx(int ordinal, std::size_t chunk) {
        fvb_ok(fvb_ctx_create(ordinal, chunk, &c), "fvb_ctx_create");
    }
    ~Ctx() { fvb_ctx_destroy(c); }
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;
};

void download(const DeviceVector& d, DenseVector& h) { d.download(h); }

// The harness runs on be.ordinal and gives the caller's thread its current
// device back on every exit.
struct OnDevice {
    int prev = -1;
    explicit OnDevice(int dev) {
        cuda_ok(cudaGetDevice(&prev), "cudaGetDevice");
        cuda_ok(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~OnDevice() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

std::string bench_label(const DeviceBackend& be) {
    return "b200x" + std::to_string(be.ordinals.empty() ? 1 : be.ordinals.size());
}

std::vector<BenchRecord> run_micro(const BenchConfig& cfg, const DeviceBackend& be,
                                   BenchPlanes where) {
    cfg.validate();
    std::vector<BenchRecord> out;
    OnDevice on(be.ordinal);
    const cudaStream_t stream = static_cast<cudaStream_t>(be.stream);
    const uint8_t prec = cfg.precision == Precision::f64 ? FVB_F64 : FVB_F32;

    for (std::size_t n : cfg.sizes) {
        Profile f = make_profile(n, cfg.precision);
        StateSet u = state_conservative(EosSpec(), 3, f.rho, f.mx, f.my, f.mz, f.rho_E);
        Expr expr = derived_v_mag2(u);
        DenseVector y(cfg.precision, n), y_hand(cfg.precision, n), y_ref(cfg.precision, n);

        std::unique_ptr<Resident> rs;
        DeviceVector yd, yd_hand;
        std::unique_ptr<Ctx> ctx;
        fvb_kernel k{};
        std::vector<void*> hargs;
        std::vector<uint8_t> hprec;
        DeviceBackend gb = be;
        if (where == BenchPlanes::Device) {
            rs = std::make_unique<Resident>(f);
            gb.residency = &rs->res;
            yd = make_temp(cfg.precision, n);
            yd_hand = make_temp(cfg.precision, n);
        } else {
            // the hand path: the same key's kernel resolved once, launched
            // over the host planes through the staged executor
            ctx = std::make_unique<Ctx>(be.ordinal, be.chunk_points);
            const std::string key = structural_key(expr, cfg.precision);
            fvb_ok(fvb_lookup(key.c_str(), &k), "fvb_lookup");
            std::vector<const DenseVector*> leaves;
            (void)block_key({expr}, {cfg.precision}, 1, 1, &leaves);
            hargs.push_back(y_hand.raw());
            for (const DenseVector* l : leaves) hargs.push_back(const_cast<void*>(l->raw()));
            hprec.assign(hargs.size(), prec);
        }
        const void* const* dev_in = nullptr;
        std::vector<const void*> dptr;
        if (rs) {
            dptr = rs->ptrs();
            dev_in = dptr.data();
        }

        auto generic = [&] {
            if (where == BenchPlanes::Device)
                evaluate(gb, expr, yd);
            else
                evaluate(gb, expr, y);
        };
        auto hand = [&] {
            if (where == BenchPlanes::Device) {
                fvb_ok(fvb_v_mag2(3, prec, n, dev_in, yd_hand.data(), stream), "fvb_v_mag2");
                cuda_ok(cudaStreamSynchronize(stream), "hand v_mag2");
            } else {
                fvb_ok(fvb_launch_host(ctx->c, &k, n, hargs.data(), hprec.data(), nullptr,
                                       nullptr, nullptr),
                       "fvb_launch_host");
            }
        };

        // warm-up, also the bitwise checks
        generic();
        hand();
        if (where == BenchPlanes::Device) {
            download(yd, y);
            download(yd_hand, y_hand);
        }
        if (!same_bits(y, y_hand))
            throw OracleMismatch("micro (device): generic and hand-fused results differ at n=" +
                                 std::to_string(n));
        fusevec::evaluate(Backend::scalar_ref(), expr, y_ref);
        if (!same_bits(y, y_ref))
            throw OracleMismatch("micro (device): device and scalar_ref results differ at n=" +
                                 std::to_string(n));

        const int reps = decide_reps(cfg, time_ns(generic) + time_ns(hand));
        std::vector<double> tg, th;
        tg.reserve(reps);
        th.reserve(reps);
        const std::uint64_t alloc0 = vector_alloc_count();
        for (int r = 0; r < reps; ++r) {  // interleaved ABAB
            tg.push_back(time_ns(generic));
            th.push_back(time_ns(hand));
        }
        check_no_alloc(alloc0, "micro");

        const double med_g = median(tg), med_h = median(th);
        BenchRecord r;
        r.suite = "micro";
        r.backend = bench_label(be) + (where == BenchPlanes::Host ? "-host" : "");
        r.precision = cfg.precision;
        r.n = n;
        r.median_ns = med_g;
        // bench.cpp:196-200: 6 flops, 5 reads + 1 write per element
        r.mflops = 6.0 * static_cast<double>(n) / med_g * 1000.0;
        r.bandwidth_mbs =
            6.0 * static_cast<double>(n * scalar_width(cfg.precision)) / med_g * 1000.0;
        r.overhead_ratio = med_g / med_h;
        r.reps = reps;
        out.push_back(std::move(r));
    }
    return out;
}

std::vector<BenchRecord> run_miniapp(const BenchConfig& cfg, const DeviceBackend& be,
                                     BenchPlanes where) {
    cfg.validate();
    std::vector<BenchRecord> out;
    OnDevice on(be.ordinal);
    const cudaStream_t stream = static_cast<cudaStream_t>(be.stream);
    const uint8_t prec = cfg.precision == Precision::f64 ? FVB_F64 : FVB_F32;

    for (std::size_t n : cfg.sizes) {
        Profile f = make_profile(n, cfg.precision);
        StateSet u = state_conservative(EosSpec(), 3, f.rho, f.mx, f.my, f.mz, f.rho_E);
        BlockExpr flux = inviscid_flux(u);
        BlockVectorGrid dest(5, 3, cfg.precision, n);
        BlockVectorGrid dest_hand(5, 3, cfg.precision, n);

        std::unique_ptr<Resident> rs;
        std::vector<DeviceVector> od, od_hand;
        Tie tie;
        std::vector<void*> dout, hout;
        std::unique_ptr<Ctx> ctx;
        DeviceBackend gb = be;
        std::vector<const void*> in;
        if (where == BenchPlanes::Device) {
            rs = std::make_unique<Resident>(f);
            gb.residency = &rs->res;
            for (int i = 0; i < 15; ++i) {
                od.push_back(make_temp(cfg.precision, n));
                od_hand.push_back(make_temp(cfg.precision, n));
            }
            for (auto& o : od) tie.dests.push_back(&o);
            for (auto& o : od_hand) dout.push_back(o.data());
            in = rs->ptrs();
        } else {
            ctx = std::make_unique<Ctx>(be.ordinal, be.chunk_points);
            for (const DenseVector* v : {&f.rho, &f.mx, &f.my, &f.mz, &f.rho_E})
                in.push_back(v->raw());
            for (std::size_t i = 0; i < 15; ++i) hout.push_back(dest_hand.get(i).raw());
        }

        auto generic = [&] {
            if (where == BenchPlanes::Device)
                evaluate_block(gb, flux, tie);
            else
                evaluate_block(gb, flux, dest);
        };
        auto hand = [&] {
            if (where == BenchPlanes::Device) {
                fvb_ok(fvb_flux(nullptr, 3, prec, n, in.data(), dout.data(), stream), "fvb_flux");
                cuda_ok(cudaStreamSynchronize(stream), "hand flux");
            } else {
                fvb_ok(fvb_flux_host(ctx->c, nullptr, 3, prec, n, in.data(), hout.data()),
                       "fvb_flux_host");
            }
        };

        generic();
        hand();
        if (where == BenchPlanes::Device)
            for (std::size_t i = 0; i < 15; ++i) {
                download(od[i], dest.get(i));
                download(od_hand[i], dest_hand.get(i));
            }

        // the reference's oracle check once per size (bench.cpp:321-336)
        const double tol = cfg.precision == Precision::f64 ? 1e-12 : 1e-6;
        for (std::size_t r = 0; r < 5; ++r)
            for (std::size_t c = 0; c < 3; ++c)
                for (std::size_t i = 0; i < n; i += (n > 256 ? n / 256 : 1)) {
                    const double want = flux_oracle(f, r, c, i);
                    const double got = dest.item(r, c).at(i);
                    const double scale = std::max(1.0, std::fabs(want));
                    if (std::fabs(got - want) > tol * scale)
                        throw OracleMismatch("miniapp (device): flux(" + std::to_string(r) + "," +
                                             std::to_string(c) + ")[" + std::to_string(i) +
                                             "] = " + std::to_string(got) + ", oracle " +
                                             std::to_string(want));
                }
        // bitwise: generic == hand == the reference's scalar backend
        {
            BlockVectorGrid dest_ref(5, 3, cfg.precision, n);
            fusevec::evaluate_block(Backend::scalar_ref(), flux, dest_ref);
            for (std::size_t i = 0; i < 15; ++i) {
                if (!same_bits(dest.get(i), dest_hand.get(i)))
                    throw OracleMismatch("miniapp (device): generic and hand-fused differ at n=" +
                                         std::to_string(n));
                if (!same_bits(dest.get(i), dest_ref.get(i)))
                    throw OracleMismatch("miniapp (device): device and scalar_ref differ at n=" +
                                         std::to_string(n));
            }
        }

        // accounting from the trees themselves (bench.cpp:347-357)
        double flops_per_elem = 0, bytes_per_elem = 0;
        for (std::size_t i = 0; i < 15; ++i) {
            const Expr e = flux.get(i).as_expr();
            flops_per_elem += static_cast<double>(count_ops(e.node()));
            std::set<const DenseVector*> leaves;
            collect_leaves(e.node(), leaves);
            bytes_per_elem +=
                static_cast<double>((leaves.size() + 1) * scalar_width(cfg.precision));
        }

        const int reps = decide_reps(cfg, time_ns(generic) + time_ns(hand));
        std::vector<double> tg, th;
        tg.reserve(reps);
        th.reserve(reps);
        const std::uint64_t alloc0 = vector_alloc_count();
        for (int r = 0; r < reps; ++r) {
            tg.push_back(time_ns(generic));
            th.push_back(time_ns(hand));
        }
        check_no_alloc(alloc0, "miniapp");

        const double med_g = median(tg), med_h = median(th);
        BenchRecord r;
        r.suite = "miniapp";
        r.backend = bench_label(be) + (where == BenchPlanes::Host ? "-host" : "");
        r.precision = cfg.precision;
        r.n = n;
        r.median_ns = med_g;
        r.mflops = flops_per_elem * static_cast<double>(n) / med_g * 1000.0;
        r.bandwidth_mbs = bytes_per_elem * static_cast<double>(n) / med_g * 1000.0;
        r.overhead_ratio = med_g / med_h;
        r.reps = reps;
        out.push_back(std::move(r));
    }
    return out;
}

}  // namespace device
}  // namespace fusevec
