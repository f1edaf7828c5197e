// integrated_api -- the reference with INTEGRATION.md §1-3 applied
// (integrate_reference.py): a user switches to the device by passing
// Backend::device() to the reference's own evaluate / evaluate_block, and
// nothing else changes.  Every result is compared with the same call on
// Backend::scalar_ref(): bitwise for +,-,*,/,sqrt, within 4 ulp for sin.
// Built in the reference's own namespace (no -Dfusevec=fvref rename).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "fusevec/backend.hpp"
#include "fusevec/bench.hpp"
#include "fusevec/block.hpp"
#include "fusevec/fluid.hpp"
#include "fusevec/rng.hpp"
#include "fusevec_device.hpp"

using namespace fusevec;

namespace {

int failures = 0;

void check(const std::string& name, const std::function<std::string()>& fn) {
    try {
        const std::string d = fn();
        std::printf("[PASS] %s%s%s\n", name.c_str(), d.empty() ? "" : ": ", d.c_str());
    } catch (const std::exception& e) {
        std::printf("[FAIL] %s: %s\n", name.c_str(), e.what());
        ++failures;
    }
    std::fflush(stdout);
}

[[noreturn]] void fail(const std::string& m) { throw std::runtime_error(m); }

bool same_bits(const DenseVector& a, const DenseVector& b) {
    return a.precision() == b.precision() && a.size() == b.size() &&
           (a.size() == 0 || std::memcmp(a.raw(), b.raw(), a.byte_size()) == 0);
}

// random_state of proj/tests/acceptance.cpp:214-230
std::vector<DenseVector> random_state(std::size_t dim, std::size_t n, SplitMix64& rng,
                                      Precision prec) {
    std::vector<DenseVector> f(dim + 2, DenseVector(prec, n));
    for (std::size_t i = 0; i < n; ++i) {
        const double rho = rng.uniform(0.5, 2.0), p = rng.uniform(0.5, 2.0);
        double vsq = 0;
        f[0].set(i, rho);
        for (std::size_t j = 0; j < dim; ++j) {
            const double v = rng.uniform(-1.0, 1.0);
            vsq += v * v;
            f[1 + j].set(i, rho * v);
        }
        f[dim + 1].set(i, p / 0.4 + 0.5 * rho * vsq);
    }
    return f;
}

StateSet state_of(std::vector<DenseVector>& f, std::size_t dim) {
    std::vector<Expr> lv;
    for (auto& v : f) lv.push_back(leaf(v));
    return state_conservative(EosSpec(), dim, lv);
}

}  // namespace

int main() {
    const Backend dev = Backend::device(), ref = Backend::scalar_ref();
    check("Backend::device() is the new kind", [&] {
        if (dev.kind() != BackendKind::Device) fail("kind");
        return "";
    });
    for (Precision P : {Precision::f64, Precision::f32}) {
        const char* pn = P == Precision::f64 ? "f64" : "f32";
        check(std::string("evaluate_block(Backend::device(), inviscid_flux(u), grid), d = 1..3, ") + pn,
              [&] {
                  SplitMix64 rng(0xD1);
                  for (std::size_t d = 1; d <= 3; ++d) {
                      const std::size_t n = 100003;
                      auto f = random_state(d, n, rng, P);
                      StateSet u = state_of(f, d);
                      BlockVectorGrid got(d + 2, d, P, n), want(d + 2, d, P, n);
                      evaluate_block(dev, inviscid_flux(u), got);
                      evaluate_block(ref, inviscid_flux(u), want);
                      for (std::size_t i = 0; i < (d + 2) * d; ++i)
                          if (!same_bits(got.get(i), want.get(i)))
                              fail("d=" + std::to_string(d) + " item " + std::to_string(i));
                  }
                  return "bitwise";
              });
        check(std::string("evaluate(Backend::device(), ...): pressure, v^2, conversion, c; ") + pn, [&] {
            SplitMix64 rng(0xD2);
            const std::size_t n = 70001;
            auto f = random_state(3, n, rng, P);
            StateSet u = state_of(f, 3);
            const std::vector<Expr> es{derived_p(u), derived_v_mag2(u), derived_c(u),
                                       convert(u, Formulation::Primitive).field(2)};
            for (const Expr& e : es) {
                DenseVector got(P, n), want(P, n);
                evaluate(dev, e, got);
                evaluate(ref, e, want);
                if (!same_bits(got, want)) fail("an expression differs");
            }
            // the member form routes the same way
            DenseVector got(P, n), want(P, n);
            dev.evaluate(derived_p(u), got);
            ref.evaluate(derived_p(u), want);
            if (!same_bits(got, want)) fail("Backend::evaluate member");
            return "bitwise";
        });
        check(std::string("evaluate_block(Backend::device(), inviscid_flux_jacobian(u)) and the CFL; ") + pn,
              [&] {
                  SplitMix64 rng(0xD3);
                  const std::size_t n = 20011;
                  auto f = random_state(3, n, rng, P);
                  StateSet u = state_of(f, 3);
                  BlockVectorGrid got(15, 5, P, n), want(15, 5, P, n);
                  evaluate_block(dev, inviscid_flux_jacobian(u), got);
                  evaluate_block(ref, inviscid_flux_jacobian(u), want);
                  for (std::size_t i = 0; i < 75; ++i)
                      if (!same_bits(got.get(i), want.get(i))) fail("item " + std::to_string(i));
                  DenseVector lam(P, n);
                  evaluate(ref, wave_speed(u), lam);
                  double mx = 0;
                  for (std::size_t i = 0; i < n; ++i) mx = std::max(mx, lam.at(i));
                  device::DeviceBackend be;
                  if (device::reduce_max(be, wave_speed(u)) != mx) fail("CFL maximum");
                  return "bitwise, CFL maximum exact";
              });
    }
    check("the paper's y = 0.5*sin(x+y) through Backend::device(), in place", [&] {
        SplitMix64 rng(1);
        const std::size_t n = 1000000;
        DenseVector x(Precision::f64, n), y(Precision::f64, n);
        for (std::size_t i = 0; i < n; ++i) x.set(i, rng.uniform(0.25, 4.0));
        for (std::size_t i = 0; i < n; ++i) y.set(i, rng.uniform(0.25, 4.0));
        DenseVector y_ref = y;
        evaluate(dev, constant(0.5, leaf(y)) * elem_sin(leaf(x) + leaf(y)), y);
        evaluate(ref, constant(0.5, leaf(y_ref)) * elem_sin(leaf(x) + leaf(y_ref)), y_ref);
        std::int64_t worst = 0;
        for (std::size_t i = 0; i < n; ++i) {
            std::int64_t a, b;
            const double va = y.at(i), vb = y_ref.at(i);
            std::memcpy(&a, &va, 8);
            std::memcpy(&b, &vb, 8);
            worst = std::max<std::int64_t>(worst, a > b ? a - b : b - a);
        }
        if (worst > 4) fail("max ulp " + std::to_string(worst));
        return "max " + std::to_string(worst) + " ulp";
    });
    check("the reference's error types through Backend::device()", [&] {
        DenseVector a(Precision::f64, 10), b(Precision::f64, 11), c(Precision::f64, 10);
        int caught = 0;
        try {
            evaluate(dev, leaf(a) + leaf(b), a);
        } catch (const LengthMismatch&) {
            ++caught;
        }
        try {
            evaluate(dev, tag(1, leaf(a)) + tag(1, leaf(c)), a);
        } catch (const TagConflict&) {
            ++caught;
        }
        if (caught != 2) fail("errors not raised");
        return "LengthMismatch, TagConflict";
    });
    check("the reference's own run_micro / run_miniapp with BenchConfig::backend = Device", [&] {
        // its harness keeps its own checks: micro bitwise generic == hand-fused
        // loop, miniapp the flux oracle and device == parallel bit for bit
        // (bench.cpp:172-176, 321-345); overhead_ratio here is the device call
        // over the reference's single-thread CPU loop
        std::string out;
        for (const char* suite : {"micro", "miniapp"}) {
            BenchConfig cfg;
            cfg.suite = suite;
            cfg.backend = BackendKind::Device;
            cfg.sizes = {1024, 65536, 1u << 20};
            cfg.reps = 3;
            const auto recs = std::string(suite) == "micro" ? run_micro(cfg) : run_miniapp(cfg);
            for (const auto& r : recs) {
                if (r.backend != "b200x1") fail("backend label " + r.backend);
                char buf[96];
                std::snprintf(buf, sizeof buf, "%s n=%zu %.3g; ", suite, r.n, r.overhead_ratio);
                out += buf;
            }
        }
        return "device / CPU hand-fused time: " + out;
    });
    std::printf(failures ? "%d check(s) failed\n" : "all checks passed\n", failures);
    return failures ? 1 : 0;
}
