// device_acceptance.cpp -- the reference's own API driving the B200 backend.
//
// Built by tests/native/Makefile against the UNMODIFIED reference (compiled
// as namespace fvref from /root/reference; test-only linkage) plus the
// product adapter paper_1809_09851_b200/host/fusevec_device.cpp and
// libfvb.so.  Mirrors the reference's acceptance criteria on the hot path
// (proj/tests/acceptance.cpp) with the device backend in place of
// Backend::scalar_ref(), comparing bit for bit against the reference engine.
//
//   device_acceptance keys   -- CPU only: structural keys of the reference's
//                               trees resolve to the fused kernels; the new
//                               fluid objects evaluate, on the reference
//                               engine, to the oracle composition
//   device_acceptance gpu    -- the device path itself
//
// Each check prints [PASS]/[FAIL]; the exit code counts failures.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
#include <chrono>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "fusevec/block.hpp"
#include "fusevec/fluid.hpp"
#include "fusevec/rng.hpp"
#include "fusevec_device.hpp"
#include "fvb.h"
#include "fvb_oracle.h"
#include "oracle.hpp"  // the reference's own test oracle/TreeGen (proj/tests/oracle.hpp)

using namespace fvref;
namespace dev = fvref::device;

namespace {

int failures = 0;

void check(const std::string& name, const std::function<std::string()>& fn) {
    try {
        std::string d = fn();
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
                                      Precision prec = Precision::f64) {
    std::vector<DenseVector> f(dim + 2, DenseVector(prec, n));
    for (std::size_t i = 0; i < n; ++i) {
        double rho = rng.uniform(0.5, 2.0);
        double p = rng.uniform(0.5, 2.0);
        double vsq = 0;
        f[0].set(i, rho);
        for (std::size_t j = 0; j < dim; ++j) {
            double v = rng.uniform(-1.0, 1.0);
            vsq += v * v;
            f[1 + j].set(i, rho * v);
        }
        f[dim + 1].set(i, p / 0.4 + 0.5 * rho * vsq);
    }
    return f;
}

std::vector<Expr> leaves_of(const std::vector<DenseVector>& vs) {
    std::vector<Expr> out;
    for (const auto& v : vs) out.push_back(leaf(v));
    return out;
}

std::string lookup_name(const std::string& key) {
    fvb_kernel k;
    if (fvb_lookup(key.c_str(), &k) != FVB_OK) return "";
    return k.name;
}

std::vector<Expr> block_items(const BlockExpr& b) {
    std::vector<Expr> items;
    for (std::size_t r = 0; r < b.block_rows(); ++r)
        for (std::size_t c = 0; c < b.block_cols(); ++c) items.push_back(b.item(r, c).as_expr());
    return items;
}

std::string block_key_of(const BlockExpr& b, Precision p) {
    auto items = block_items(b);
    std::vector<Precision> dests(items.size(), p);
    return dev::block_key(items, dests, b.block_rows(), b.block_cols(), nullptr);
}

// ---------------------------------------------------------------------------
// keys: CPU only
// ---------------------------------------------------------------------------

void run_keys() {
    for (Precision P : {Precision::f64, Precision::f32}) {
        const std::string sfx = P == Precision::f64 ? "_f64" : "_f32";
        for (std::size_t d = 1; d <= 3; ++d) {
            const std::string tag = std::to_string(d) + sfx;
            check("keys: reference trees resolve, d" + tag, [&] {
                SplitMix64 rng(1);
                auto f = random_state(d, 4, rng, P);
                StateSet u = state_conservative(EosSpec(), d, leaves_of(f));
                struct Case {
                    std::string want, key;
                };
                BlockExpr prim = convert(u, Formulation::Primitive).block();
                std::vector<Expr> prim_items = block_items(prim);
                prim_items.erase(prim_items.begin());  // rho passes through
                std::vector<Expr> with_c = prim_items;
                with_c.push_back(derived_c(u));
                std::vector<Precision> pd(with_c.size(), P);
                std::vector<Case> cases = {
                    {"flux" + tag, block_key_of(inviscid_flux(u), P)},
                    {"jacobian" + tag, block_key_of(inviscid_flux_jacobian(u), P)},
                    {"cons2prim" + tag, dev::block_key(prim_items, std::vector<Precision>(d + 1, P),
                                                       d + 1, 1, nullptr)},
                    {"cons2prim_c" + tag, dev::block_key(with_c, pd, d + 2, 1, nullptr)},
                    {"pressure" + tag, dev::structural_key(derived_p(u), P)},
                    {"sound_speed" + tag, dev::structural_key(derived_c(u), P)},
                    {"v_mag2" + tag, dev::structural_key(derived_v_mag2(u), P)},
                    {"wave_speed" + tag, dev::structural_key(wave_speed(u), P)},
                };
                StateSet w = state_primitive(EosSpec(), d, leaves_of(f));
                std::vector<Expr> cons_items = block_items(convert(w, Formulation::Conservative).block());
                cons_items.erase(cons_items.begin());
                cases.push_back({"prim2cons" + tag, dev::block_key(cons_items,
                                                                   std::vector<Precision>(d + 1, P),
                                                                   d + 1, 1, nullptr)});
                cases.push_back({"flux_prim" + tag, block_key_of(inviscid_flux(w), P)});
                for (const Case& c : cases)
                    if (lookup_name(c.key) != c.want)
                        fail(c.want + " not resolved from key " + c.key.substr(0, 120));
                // a non-default gas resolves to the same kernels
                StateSet mono = state_conservative(EosSpec(rational(5, 2), rational(3, 2)), d,
                                                   leaves_of(f));
                if (lookup_name(block_key_of(inviscid_flux(mono), P)) != "flux" + tag)
                    fail("monatomic flux key not resolved");
                return std::to_string(cases.size() + 1) + " trees";
            });
        }
        check("new fluid objects on the reference engine == C oracle" + sfx, [&] {
            // The product's derived_c / wave_speed / inviscid_flux_jacobian
            // (fusevec_device.cpp), evaluated by the UNMODIFIED reference
            // engine, reproduce oracle/fvb_oracle.c bit for bit.
            for (std::size_t d = 1; d <= 3; ++d) {
                SplitMix64 rng(77 + d);
                const std::size_t n = 513;
                auto f = random_state(d, n, rng, P);
                StateSet u = state_conservative(EosSpec(), d, leaves_of(f));
                const std::size_t w = d + 2;
                BlockVectorGrid J(d * w, w, P, n);
                evaluate_block(Backend::scalar_ref(), inviscid_flux_jacobian(u), J);
                DenseVector c(P, n), lam(P, n);
                evaluate(Backend::scalar_ref(), derived_c(u), c);
                evaluate(Backend::scalar_ref(), wave_speed(u), lam);
                std::vector<DenseVector> oj(d * w * w, DenseVector(P, n)), oc(d + 2, DenseVector(P, n));
                std::vector<const void*> in;
                for (auto& v : f) in.push_back(v.raw());
                std::vector<void*> jo, co;
                for (auto& v : oj) jo.push_back(v.raw());
                for (auto& v : oc) co.push_back(v.raw());
                fvo_gas g = fvo_default_gas();
                if (P == Precision::f64) {
                    fvo_jacobian_f64(g, int(d), n, (const double* const*)in.data(), (double* const*)jo.data(), nullptr);
                    fvo_cons2prim_f64(g, int(d), n, (const double* const*)in.data(), (double* const*)co.data());
                } else {
                    fvo_jacobian_f32(g, int(d), n, (const float* const*)in.data(), (float* const*)jo.data(), nullptr);
                    fvo_cons2prim_f32(g, int(d), n, (const float* const*)in.data(), (float* const*)co.data());
                }
                for (std::size_t i = 0; i < d * w * w; ++i)
                    if (!same_bits(J.get(i), oj[i])) fail("jacobian item " + std::to_string(i));
                if (!same_bits(c, oc[d + 1])) fail("sound speed");
                double m = 0;
                for (std::size_t i = 0; i < n; ++i) m = std::fmax(m, lam.at(i));
                double om = P == Precision::f64 ? fvo_wave_speed_max_f64(g, int(d), n, (const double* const*)in.data())
                                                : double(fvo_wave_speed_max_f32(g, int(d), n, (const float* const*)in.data()));
                if (m != om) fail("wave speed max");
            }
            return "d = 1, 2, 3";
        });
        check("keys: axpy-sin and EOS" + sfx, [&] {
            DenseVector x(P, 4), y(P, 4);
            Expr e = constant(0.5, leaf(y)) * elem_sin(leaf(x) + leaf(y));
            if (lookup_name(dev::structural_key(e, P)) != "axpy_sin" + sfx) fail("axpy-sin");
            Expr et = tag(0, leaf(x));  // tags are transparent to the key
            Expr e2 = constant(0.5, leaf(y)) * elem_sin(et + tag(1, leaf(y)));
            if (lookup_name(dev::structural_key(e2, P)) != "axpy_sin" + sfx) fail("tagged axpy");
            IdealGasEos gas;
            if (lookup_name(dev::structural_key(gas.p_rhoe(leaf(x), leaf(y)), P)) != "eos_p" + sfx)
                fail("eos_p");
            if (lookup_name(dev::structural_key(gas.T_rhoe(leaf(x), leaf(y)), P)) != "eos_T" + sfx)
                fail("eos_T");
            // a tree with no hand-written kernel is lowered (or, without a
            // device, not loaded) -- never matched to a fused pattern
            const std::string nm = lookup_name(dev::structural_key(elem_cos(leaf(x)), P));
            if (!nm.empty() && nm.rfind("gen:", 0) != 0) fail("cos matched " + nm);
            return "";
        });
    }
}

// ---------------------------------------------------------------------------
// gpu: the device path
// ---------------------------------------------------------------------------

void run_gpu() {
    dev::DeviceBackend be;
    Backend ref = Backend::scalar_ref();

    check("criterion 1 on device: zero overhead, the reference's gate (acceptance.cpp:46-62)", [&] {
        // run_micro at n = 2^20, auto reps: the reference's tree through
        // evaluate() against the fused kernel called directly; the harness
        // itself checks both against scalar_ref bit for bit
        const double gate = 1.10;
        double ratio[2], mini[2];
        const Precision precs[2] = {Precision::f64, Precision::f32};
        for (int k = 0; k < 2; ++k) {
            BenchConfig cfg;
            cfg.sizes = {1u << 20};
            cfg.reps = 0;
            cfg.precision = precs[k];
            cfg.suite = "micro";
            ratio[k] = dev::run_micro(cfg, be).at(0).overhead_ratio;
            cfg.suite = "miniapp";
            mini[k] = dev::run_miniapp(cfg, be).at(0).overhead_ratio;
        }
        char buf[200];
        std::snprintf(buf, sizeof buf,
                      "n=2^20 micro ratios f64 %.4f, f32 %.4f (gate %.2f); miniapp f64 %.4f, f32 %.4f",
                      ratio[0], ratio[1], gate, mini[0], mini[1]);
        if (ratio[0] > gate || ratio[1] > gate) fail(buf);
        return std::string(buf);
    });

    check("criterion 4 on device: backend equivalence on random trees (acceptance.cpp:161-205)", [&] {
        // The reference's criterion: TreeGen trees of depth 5 with tagged
        // leaves over mixed f32/f64 pools of lengths 1, 2, 257 and 1024
        // (tree t on length t % 4), each evaluated by two backends.  Here the
        // device backend against scalar_ref: trees of exact ops bit for bit,
        // trees with libm nodes within rtol 1e-3 on every element of these
        // short vectors (a few-ulp libm difference, propagated).  1000 trees
        // as in the reference with FVB_ACC_C4_TREES=1000 (every distinct
        // tree is one NVRTC compile; the default keeps the suite short).
        const std::size_t lens[4] = {1, 2, 257, 1024};
        std::vector<std::vector<DenseVector>> pools(4);
        SplitMix64 seed_rng(0xACCE55);
        for (int k = 0; k < 4; ++k) {
            pools[k].push_back(testutil::make_vec(Precision::f64, lens[k], seed_rng));
            pools[k].push_back(testutil::make_vec(Precision::f32, lens[k], seed_rng));
            pools[k].push_back(testutil::make_vec(Precision::f64, lens[k], seed_rng));
        }
        const char* nt = std::getenv("FVB_ACC_C4_TREES");
        const int trees = nt && *nt ? std::atoi(nt) : 120;
        SplitMix64 rng(0xE0E0);
        int exact = 0, approx = 0, constant = 0;
        for (int t = 0; t < trees; ++t) {
            const int k = t % 4;
            const std::size_t n = lens[k];
            testutil::TreeGen gen{&pools[k], true};
            Expr e = gen.gen(rng, 5);
            const Precision P = e.result_precision();
            DenseVector want(P, n), got(P, n);
            evaluate(ref, e, want);
            try {
                dev::evaluate(be, e, got);
            } catch (const UnsupportedExpression&) {
                // a leafless tree with a non-finite constant: the reference's
                // JIT refuses it too (backend_jit.cpp:323-334)
                ++constant;
                continue;
            }
            const std::string key = dev::structural_key(e, P);
            bool lib = false;
            for (std::size_t i = 0; i + 1 < key.size(); ++i) {
                if (key[i] != 'U' && key[i] != 'B') continue;
                char* end = nullptr;
                const long op = std::strtol(key.c_str() + i + 1, &end, 10);
                if (!end || (*end != 's' && *end != 'd')) continue;
                lib = lib || (key[i] == 'U' ? ((op >= 2 && op <= 14) || op == 16 || op == 20)
                                            : (op == 4 || op == 7));
            }
            if (!lib) {
                ++exact;
                if (!same_bits(want, got)) fail("tree " + std::to_string(t) + " differs bitwise: " +
                                                key.substr(0, 120));
                continue;
            }
            ++approx;
            for (std::size_t i = 0; i < n; ++i)
                if (!testutil::scalar_close(want.at(i), got.at(i), 1e-3) &&
                    !(std::isnan(want.at(i)) && std::isnan(got.at(i))))
                    fail("tree " + std::to_string(t) + " element " + std::to_string(i) + ": " +
                         std::to_string(want.at(i)) + " vs " + std::to_string(got.at(i)) + " " +
                         key.substr(0, 120));
        }
        return std::to_string(trees) + " trees (lengths 1/2/257/1024, tagged leaves, depth 5): " +
               std::to_string(exact) + " exact-op trees bitwise, " + std::to_string(approx) +
               " libm trees within rtol 1e-3" +
               (constant ? ", " + std::to_string(constant) + " refused as non-finite constants"
                         : std::string());
    });

    check("criterion 8 on device: the benchmark CSV emitter (acceptance.cpp:404-421)", [&] {
        BenchConfig cfg;
        cfg.suite = "micro";
        cfg.sizes = {1024};
        cfg.reps = 3;
        auto recs = dev::run_micro(cfg, be);
        std::ostringstream os;
        write_csv(recs, os);
        const std::string text = os.str();
        if (text.find("suite,backend,precision,n,median_ns,mflops,bandwidth_mbs,overhead_ratio\n") ==
            std::string::npos)
            fail("CSV header missing");
        if (text.find("micro,b200x1,f64,1024,") == std::string::npos) fail("CSV row missing");
        return "the reference's write_csv over device records: header and micro,b200x1,f64,1024 row";
    });

    check("general lowering: random trees (the reference's TreeGen) vs scalar_ref", [&] {
        // proj/tests/test_backend.cpp:267-290 checks its compiled path on
        // TreeGen trees at n=16384; here the device path (fvb_lookup's NVRTC
        // lowering) on the same kind of trees.  Trees of exact ops only
        // (+ - * / sqrt abs neg ceil floor round min max) must match bit
        // for bit; trees with libm functions within rtol 1e-9 when every
        // libm node is f64, 1e-5 when one is f32 (scalar_close of
        // oracle.hpp) on at least 99.9% of elements: CUDA's and glibc's
        // transcendentals differ by a few ulp of the node's precision.
        std::vector<DenseVector> pool;
        SplitMix64 seed_rng(661);
        const std::size_t n = 16384;
        pool.push_back(testutil::make_vec(Precision::f64, n, seed_rng));
        pool.push_back(testutil::make_vec(Precision::f32, n, seed_rng));
        pool.push_back(testutil::make_vec(Precision::f64, n, seed_rng));
        testutil::TreeGen gen{&pool, false};
        SplitMix64 rng(662);
        int exact = 0, approx = 0;
        std::size_t worst = 0;
        // FVB_ACC_TREES / FVB_ACC_DEPTH widen the sweep for stress runs
        const char* nt = std::getenv("FVB_ACC_TREES");
        const char* nd = std::getenv("FVB_ACC_DEPTH");
        const int trees = nt && *nt ? std::atoi(nt) : 80;
        const int depth = nd && *nd ? std::atoi(nd) : 4;
        for (int t = 0; t < trees; ++t) {
            Expr e = gen.gen(rng, depth);
            const Precision P = e.result_precision();
            DenseVector want(P, n), got(P, n);
            evaluate(ref, e, want);
            dev::evaluate(be, e, got);
            const std::string key = dev::structural_key(e, P);
            // libm nodes and their precisions (op codes: expr.hpp:12-46)
            bool tr32 = false, tr64 = false;
            for (std::size_t i = 0; i + 1 < key.size(); ++i) {
                if (key[i] != 'U' && key[i] != 'B') continue;
                char* end = nullptr;
                const long op = std::strtol(key.c_str() + i + 1, &end, 10);
                if (!end || (*end != 's' && *end != 'd')) continue;
                const bool lib = key[i] == 'U' ? ((op >= 2 && op <= 14) || op == 16 || op == 20)
                                               : (op == 4 || op == 7);
                if (lib) (*end == 's' ? tr32 : tr64) = true;
            }
            if (!tr32 && !tr64) {
                ++exact;
                if (!same_bits(want, got)) fail("exact tree differs bitwise: " + key.substr(0, 120));
            } else {
                ++approx;
                // A libm difference of a few ulp propagates through the rest
                // of the tree with that tree's condition number (tan near a
                // pole amplifies it without bound), so whole libm trees only
                // guard against gross lowering errors -- a wrong op, operand
                // or conversion changes essentially every element.  The
                // per-op ulp bounds are the next check.
                std::size_t bad = 0, first = n;
                for (std::size_t i = 0; i < n; ++i)
                    if (!testutil::scalar_close(want.at(i), got.at(i), 1e-3)) {
                        if (first == n) first = i;
                        ++bad;
                    }
                worst = std::max(worst, bad);
                if (bad > n / 100) {
                    char buf[200];
                    std::snprintf(buf, sizeof buf, "%zu of %zu beyond rtol 1e-3, first at %zu: %.17g vs %.17g ",
                                  bad, n, first, want.at(first), got.at(first));
                    fail(std::string("tree ") + buf + key.substr(0, 120));
                }
            }
        }
        return std::to_string(exact) + " exact trees bitwise, " + std::to_string(approx) +
               " libm trees agree on >= 99% of elements at rtol 1e-3 (worst tree: " +
               std::to_string(worst) + " of " + std::to_string(n) + " beyond)";
    });

    check("general lowering: every libm op within its ulp bound of glibc", [&] {
        // One op per tree, so no amplification: device (CUDA libdevice via
        // NVRTC) against the reference's glibc call, max ulp over 65536
        // points.  Bounds: 4 ulp f64 (north_star: <= 4 ulp incl. sin), 8 ulp
        // f32 (CUDA's single-precision bounds are up to 4 ulp, glibc's 1).
        const std::size_t n = 65536;
        struct Op {
            const char* name;
            int op;
            bool binary;
            double lo, hi, lo2, hi2;
        };
        const Op ops[] = {{"sin", 2, false, -8, 8},      {"cos", 3, false, -8, 8},
                          {"tan", 4, false, -1.4, 1.4},  {"asin", 5, false, -0.99, 0.99},
                          {"acos", 6, false, -0.99, 0.99}, {"atan", 7, false, -8, 8},
                          {"sinh", 8, false, -5, 5},     {"cosh", 9, false, -5, 5},
                          {"tanh", 10, false, -5, 5},    {"exp", 11, false, -20, 20},
                          {"log", 12, false, 0.01, 100}, {"log2", 13, false, 0.01, 100},
                          {"log10", 14, false, 0.01, 100}, {"cbrt", 16, false, -100, 100},
                          {"erf", 20, false, -3, 3},     {"pow", 4, true, 0.1, 4, -3, 3},
                          {"atan2", 7, true, -4, 4, -4, 4}};
        std::string report;
        for (Precision P : {Precision::f64, Precision::f32}) {
            const long bound = P == Precision::f64 ? 4 : 8;
            for (const Op& o : ops) {
                SplitMix64 rng(1234 + o.op + (o.binary ? 100 : 0));
                DenseVector x(P, n), y(P, n), want(P, n), got(P, n);
                for (std::size_t i = 0; i < n; ++i) x.set(i, rng.uniform(o.lo, o.hi));
                for (std::size_t i = 0; i < n; ++i) y.set(i, rng.uniform(o.lo2, o.hi2));
                Expr e = o.binary ? binary(BinaryOp(o.op), leaf(x), leaf(y))
                                  : unary(UnaryOp(o.op), leaf(x));
                evaluate(ref, e, want);
                dev::evaluate(be, e, got);
                long worst_ulp = 0;
                for (std::size_t i = 0; i < n; ++i) {
                    long d;
                    if (P == Precision::f64) {
                        long long a, b;
                        double va = want.at(i), vb = got.at(i);
                        std::memcpy(&a, &va, 8);
                        std::memcpy(&b, &vb, 8);
                        if (a < 0) a = (long long)0x8000000000000000ULL - a;
                        if (b < 0) b = (long long)0x8000000000000000ULL - b;
                        d = long(std::llabs(a - b));
                    } else {
                        int a, b;
                        float va = float(want.at(i)), vb = float(got.at(i));
                        std::memcpy(&a, &va, 4);
                        std::memcpy(&b, &vb, 4);
                        if (a < 0) a = int(0x80000000u) - a;
                        if (b < 0) b = int(0x80000000u) - b;
                        d = std::labs(long(a) - long(b));
                    }
                    worst_ulp = std::max(worst_ulp, d);
                }
                if (worst_ulp > bound)
                    fail(std::string(o.name) + (P == Precision::f64 ? " f64: " : " f32: ") +
                         std::to_string(worst_ulp) + " ulp > " + std::to_string(bound));
                report += std::string(o.name) + (P == Precision::f64 ? "" : "f") + "=" +
                          std::to_string(worst_ulp) + " ";
            }
        }
        return "max ulp: " + report;
    });

    check("matvec operands are snapshots taken before any destination is written (block.cpp:389-411)", [&] {
        // test_block.cpp:214-230: y = [0 I; I 0] * y swaps the two vectors;
        // also items built by hand whose later operand is an earlier
        // destination, and resident operands whose plane is a destination
        SplitMix64 rng(66);
        const std::size_t n = 37;
        std::vector<Triplet> eye;
        for (std::size_t i = 0; i < n; ++i) eye.push_back({i, i, 1.0});
        const SparseMatrix zero(n, n, {}), I(n, n, eye);
        BlockMatrix swap(2, 2, zero, I, I, zero);
        auto fresh = [&] {
            std::vector<DenseVector> v;
            v.push_back(testutil::make_vec(Precision::f64, n, rng, -2.0, 2.0));
            v.push_back(testutil::make_vec(Precision::f64, n, rng, -2.0, 2.0));
            return v;
        };
        {   // host vectors
            auto v = fresh();
            const std::vector<DenseVector> old = v;
            BlockColVector want(std::vector<DenseVector>{v[0], v[1]}), got(std::move(v));
            BlockExpr pw = block_matvec(swap, want), pg = block_matvec(swap, got);
            evaluate_block(ref, pw, want);
            dev::evaluate_block(be, pg, got);
            if (!same_bits(got.get(0), old[1]) || !same_bits(got.get(1), old[0]) ||
                !same_bits(got.get(0), want.get(0)) || !same_bits(got.get(1), want.get(1)))
                fail("y = swap * y on host vectors");
        }
        {   // item 1 reads item 0's destination: it must see the old value
            auto v = fresh();
            DenseVector a = testutil::make_vec(Precision::f64, n, rng, -2.0, 2.0);
            const DenseVector old0 = v[0];
            BlockColVector got(std::move(v));
            std::vector<BlockItem> items;
            items.push_back(BlockItem(std::vector<MatVecTerm>{{&I, leaf(a)}}));
            items.push_back(BlockItem(std::vector<MatVecTerm>{{&I, leaf(got.get(0))}}));
            dev::evaluate_block(be, BlockExpr(2, 1, std::move(items)), got);
            if (!same_bits(got.get(0), a) || !same_bits(got.get(1), old0))
                fail("a later operand saw an earlier destination's new value");
        }
        {   // resident operands whose planes are the tie'd destinations
            auto v = fresh();
            const std::vector<DenseVector> old = v;
            std::vector<dev::DeviceVector> dvs;
            for (auto& x : v) {
                dvs.push_back(dev::make_temp(Precision::f64, n));
                dvs.back().upload(x);
            }
            dev::Residency res;
            res.bind(v[0], dvs[0]);
            res.bind(v[1], dvs[1]);
            dev::DeviceBackend rb;
            rb.residency = &res;
            BlockColVector yv(std::vector<DenseVector>{v[0], v[1]});
            std::vector<BlockItem> ops;
            ops.push_back(BlockItem(leaf(v[0])));
            ops.push_back(BlockItem(leaf(v[1])));
            dev::evaluate_block(rb, block_matvec(swap, BlockExpr(2, 1, std::move(ops))),
                                dev::tie(dvs[0], dvs[1]));
            DenseVector t0(Precision::f64, n), t1(Precision::f64, n);
            dvs[0].download(t0);
            dvs[1].download(t1);
            if (!same_bits(t0, old[1]) || !same_bits(t1, old[0]))
                fail("resident operands aliasing tie'd destinations");
        }
        return "";
    });

    check("blocks mixing matvec rows and element-wise items that read each other's destinations", [&] {
        // block.cpp:389-451: operands captured first, then items in order --
        // an element-wise item after a matvec row reads its new value, one
        // before it the old
        SplitMix64 rng(77);
        const std::size_t n = 29;
        std::vector<Triplet> trips;
        for (std::size_t r = 0; r < n; ++r)
            for (std::size_t c = 0; c < n; ++c)
                if (rng.uniform() < 0.3) trips.push_back({r, c, rng.uniform(-2.0, 2.0)});
        const SparseMatrix M(n, n, trips);
        auto vec = [&] { return testutil::make_vec(Precision::f64, n, rng, -2.0, 2.0); };
        DenseVector x = vec();
        for (int variant = 0; variant < 3; ++variant) {
            std::vector<DenseVector> init{vec(), vec(), vec()};
            BlockColVector want{std::vector<DenseVector>(init)}, got{std::vector<DenseVector>(init)};
            auto build = [&](BlockColVector& y) {
                std::vector<BlockItem> it;
                const Expr two = constant(2.0, Precision::f64);
                if (variant == 0) {  // after: item 1 reads the matvec's new d0
                    it.push_back(BlockItem(std::vector<MatVecTerm>{{&M, leaf(x)}}));
                    it.push_back(BlockItem(leaf(y.get(0)) * two));
                    it.push_back(BlockItem(leaf(y.get(2)) + leaf(x)));
                } else if (variant == 1) {  // before: item 0 reads d1's old value
                    it.push_back(BlockItem(leaf(y.get(1)) * two));
                    it.push_back(BlockItem(std::vector<MatVecTerm>{{&M, leaf(y.get(0))}}));
                    it.push_back(BlockItem(leaf(y.get(1)) - leaf(x)));
                } else {  // a later item reading an element-wise and a matvec destination
                    it.push_back(BlockItem(leaf(x) * two));
                    it.push_back(BlockItem(std::vector<MatVecTerm>{{&M, leaf(x)}}));
                    it.push_back(BlockItem(leaf(y.get(0)) + leaf(y.get(1))));
                }
                return BlockExpr(3, 1, std::move(it));
            };
            evaluate_block(ref, build(want), want);
            dev::evaluate_block(be, build(got), got);
            for (std::size_t i = 0; i < 3; ++i)
                if (!same_bits(got.get(i), want.get(i)))
                    fail("variant " + std::to_string(variant) + " item " + std::to_string(i));
        }
        return "";
    });

    check("criterion 7 on device: CSR block matvec, all shapes <= 3x3, dims <= 8, bitwise", [&] {
        // acceptance.cpp:343-379 builds random sparse blocks and compares to a
        // dense oracle within 1e-12; the device path must equal the
        // reference's own evaluate_block bit for bit (same summation order).
        SplitMix64 rng(0xB10C);
        int cases = 0;
        for (std::size_t br = 1; br <= 3; ++br)
            for (std::size_t bc = 1; bc <= 3; ++bc)
                for (std::size_t n = 1; n <= 8; n += 3)
                    for (std::size_t m = 1; m <= 8; m += 3) {
                        std::vector<SparseMatrix> blocks;
                        for (std::size_t i = 0; i < br * bc; ++i) {
                            std::vector<Triplet> trips;
                            for (std::size_t r = 0; r < n; ++r)
                                for (std::size_t c = 0; c < m; ++c)
                                    if (rng.uniform() < 0.5)
                                        trips.push_back({r, c, rng.uniform(-2.0, 2.0)});
                            blocks.emplace_back(n, m, trips);
                        }
                        BlockMatrix mat(br, bc, std::move(blocks));
                        std::vector<DenseVector> x;
                        std::vector<BlockItem> xi;
                        for (std::size_t c = 0; c < bc; ++c)
                            x.push_back(testutil::make_vec(Precision::f64, m, rng, -2.0, 2.0));
                        for (auto& v : x) xi.push_back(BlockItem(v));
                        BlockExpr prod = block_matvec(mat, BlockExpr(bc, 1, std::move(xi)));
                        std::vector<DenseVector> wd, gd;
                        for (std::size_t r = 0; r < br; ++r) {
                            wd.emplace_back(Precision::f64, n);
                            gd.emplace_back(Precision::f64, n);
                        }
                        BlockColVector want(std::move(wd)), got(std::move(gd));
                        evaluate_block(ref, prod, want);
                        dev::evaluate_block(be, prod, got);
                        for (std::size_t r = 0; r < br; ++r)
                            if (!same_bits(want.get(r), got.get(r))) fail("matvec differs");
                        ++cases;
                    }
        // identity blocks with expression operands (acceptance.cpp:381-395):
        // y = [I I; I I] [sin(x0+x1); cos(x0-x1)] at x = 0 is all ones
        const std::size_t n = 8;
        std::vector<Triplet> diag;
        for (std::size_t i = 0; i < n; ++i) diag.push_back({i, i, 1.0});
        SparseMatrix ident(n, n, diag);
        BlockMatrixView mv(2, 2, {&ident, &ident, &ident, &ident});
        DenseVector x0(Precision::f64, n), x1(Precision::f64, n);
        BlockExpr rhs = make_block_expr(2, 1, elem_sin(leaf(x0) + leaf(x1)),
                                        elem_cos(leaf(x0) - leaf(x1)));
        BlockColVector y({DenseVector(Precision::f64, n), DenseVector(Precision::f64, n)});
        dev::evaluate_block(be, block_matvec(mv, rhs), y);
        for (std::size_t r = 0; r < 2; ++r)
            for (std::size_t i = 0; i < n; ++i)
                if (y.get(r).at(i) != 1.0) fail("identity-blocks case is not all ones");
        // f32 destination, f64 operand: accumulation in the destination's precision
        SparseMatrix a(4, 3, {{0, 0, 0.1}, {0, 2, 0.3}, {2, 1, -0.7}, {3, 2, 1.5}}, Precision::f32);
        DenseVector xv = testutil::make_vec(Precision::f64, 3, rng);
        std::vector<DenseVector> w32, g32;
        w32.emplace_back(Precision::f32, 4);
        g32.emplace_back(Precision::f32, 4);
        BlockColVector w3(std::move(w32)), g3(std::move(g32));
        BlockExpr p32 = block_matvec(BlockMatrixView(1, 1, a), make_block_expr(1, 1, leaf(xv)));
        evaluate_block(ref, p32, w3);
        dev::evaluate_block(be, p32, g3);
        if (!same_bits(w3.get(0), g3.get(0))) fail("mixed-precision matvec differs");
        // a device-resident matrix (DeviceCsr bound in a Residency): same bits,
        // and a refreshed copy follows SparseMatrix::set_value
        dev::DeviceCsr da(a, be.ordinal);
        dev::Residency res;
        res.bind(a, da);
        dev::DeviceBackend rb = be;
        rb.residency = &res;
        std::vector<DenseVector> r32;
        r32.emplace_back(Precision::f32, 4);
        BlockColVector gr(std::move(r32));
        dev::evaluate_block(rb, p32, gr);
        if (!same_bits(w3.get(0), gr.get(0))) fail("resident-matrix matvec differs");
        a.set_value(2, 1, 0.25);
        da.upload(a);
        evaluate_block(ref, p32, w3);
        dev::evaluate_block(rb, p32, gr);
        if (!same_bits(w3.get(0), gr.get(0))) fail("refreshed resident matrix differs");
        return std::to_string(cases) +
               " random block shapes bitwise; identity case all ones; resident matrix";
    });

    check("criterion 6 on device: flux, d in {1,2,3} x 100 instances, n=64, bitwise", [&] {
        SplitMix64 rng(0xF1);
        for (std::size_t d = 1; d <= 3; ++d)
            for (int inst = 0; inst < 100; ++inst) {
                auto f = random_state(d, 64, rng);
                StateSet u = state_conservative(EosSpec(), d, leaves_of(f));
                BlockExpr flux = inviscid_flux(u);
                BlockVectorGrid want(d + 2, d, Precision::f64, 64), got(d + 2, d, Precision::f64, 64);
                evaluate_block(ref, flux, want);
                dev::evaluate_block(be, flux, got);
                for (std::size_t i = 0; i < (d + 2) * d; ++i)
                    if (!same_bits(want.get(i), got.get(i))) fail("d=" + std::to_string(d));
            }
        return "";
    });

    check("f32 flux (conservative and primitive states), conversion and sound speed on device, d = 1..3", [&] {
        SplitMix64 rng(0xF32);
        for (std::size_t d = 1; d <= 3; ++d) {
            const std::size_t n = 10007;
            auto f = random_state(d, n, rng, Precision::f32);
            StateSet u = state_conservative(EosSpec(), d, leaves_of(f));
            BlockVectorGrid want(d + 2, d, Precision::f32, n), got(d + 2, d, Precision::f32, n);
            evaluate_block(ref, inviscid_flux(u), want);
            dev::evaluate_block(be, inviscid_flux(u), got);
            for (std::size_t i = 0; i < (d + 2) * d; ++i)
                if (!same_bits(want.get(i), got.get(i))) fail("f32 flux d=" + std::to_string(d));
            StateSet w = convert(u, Formulation::Primitive);
            std::vector<DenseVector> pd;
            for (std::size_t i = 0; i < d + 2; ++i) pd.emplace_back(Precision::f32, n);
            BlockColVector pv(std::move(pd));
            dev::evaluate_block(be, w.block(), pv);
            for (std::size_t i = 0; i < d + 2; ++i) {
                DenseVector wi(Precision::f32, n);
                evaluate(ref, w.field(i), wi);
                if (!same_bits(wi, pv.get(i))) fail("f32 primitive field " + std::to_string(i));
            }
            DenseVector cw(Precision::f32, n), cg(Precision::f32, n);
            evaluate(ref, derived_c(u), cw);
            dev::evaluate(be, derived_c(u), cg);
            if (!same_bits(cw, cg)) fail("f32 sound speed d=" + std::to_string(d));
            // the flux of a primitive-formulation state (fluid.cpp:290-298)
            std::vector<Expr> pl;
            for (std::size_t i = 0; i < d + 2; ++i) pl.push_back(leaf(pv.get(i)));
            StateSet up = state_primitive(EosSpec(), d, pl);
            BlockVectorGrid fw(d + 2, d, Precision::f32, n), fg(d + 2, d, Precision::f32, n);
            evaluate_block(ref, inviscid_flux(up), fw);
            dev::evaluate_block(be, inviscid_flux(up), fg);
            for (std::size_t i = 0; i < (d + 2) * d; ++i)
                if (!same_bits(fw.get(i), fg.get(i))) fail("primitive-state flux d=" + std::to_string(d));
        }
        return "";
    });

    check("criterion 6 worked instance on device: column 0 = [2,4,4,4,16]", [&] {
        DenseVector rho({2.0}), mx({2.0}), my({4.0}), mz({4.0}), rhoE({14.0});
        StateSet u = state_conservative(EosSpec(), 3, rho, mx, my, mz, rhoE);
        BlockVectorGrid got(5, 3, Precision::f64, 1);
        dev::evaluate_block(be, inviscid_flux(u), got);
        const double want[5] = {2, 4, 4, 4, 16};
        for (std::size_t r = 0; r < 5; ++r)
            if (got.item(r, 0).at(0) != want[r]) fail("row " + std::to_string(r));
        return "";
    });

    check("criterion 5 on device: round trip and p = rho R T, 100 x d, n=128", [&] {
        SplitMix64 rng(0x7E6);
        for (std::size_t d = 1; d <= 3; ++d)
            for (int inst = 0; inst < 100; ++inst) {
                auto f = random_state(d, 128, rng);
                StateSet uc = state_conservative(EosSpec(), d, leaves_of(f));
                // cons -> prim on the device (rho passes through)
                std::vector<DenseVector> prim;
                for (std::size_t i = 0; i < d + 2; ++i) prim.emplace_back(Precision::f64, 128);
                BlockColVector pv(std::move(prim));
                dev::evaluate_block(be, convert(uc, Formulation::Primitive).block(), pv);
                // prim -> cons on the device
                std::vector<Expr> pf;
                for (std::size_t i = 0; i < d + 2; ++i) pf.push_back(leaf(pv.get(i)));
                StateSet up = state_primitive(EosSpec(), d, pf);
                std::vector<DenseVector> back;
                for (std::size_t i = 0; i < d + 2; ++i) back.emplace_back(Precision::f64, 128);
                BlockColVector bv(std::move(back));
                dev::evaluate_block(be, convert(up, Formulation::Conservative).block(), bv);
                for (std::size_t fi = 0; fi < d + 2; ++fi)
                    for (std::size_t i = 0; i < 128; ++i) {
                        double a = bv.get(fi).at(i), b = f[fi].at(i);
                        if (std::fabs(a - b) > 1e-12 * std::fmax(std::fmax(std::fabs(a), std::fabs(b)), 1.0))
                            fail("round trip drifted");
                    }
                // and the device primitive fields equal the reference's bitwise
                StateSet w = convert(uc, Formulation::Primitive);
                for (std::size_t fi = 1; fi < d + 2; ++fi) {
                    DenseVector want(Precision::f64, 128);
                    evaluate(ref, w.field(fi), want);
                    if (!same_bits(want, pv.get(fi))) fail("primitive field differs");
                }
            }
        return "";
    });

    check("fusion: zero intermediate vector allocations on the device path", [&] {
        SplitMix64 rng(3);
        auto f = random_state(3, 16384, rng);
        StateSet u = state_conservative(EosSpec(), 3, leaves_of(f));
        BlockVectorGrid grid(5, 3, Precision::f64, 16384);
        dev::evaluate_block(be, inviscid_flux(u), grid);  // warm
        const auto before = vector_alloc_count();
        dev::evaluate_block(be, inviscid_flux(u), grid);
        if (vector_alloc_count() != before) fail("DenseVector allocated");
        return "";
    });

    check("sound speed, v_mag2, pressure, EOS and axpy-sin on device, bitwise / 4 ulp", [&] {
        SplitMix64 rng(9);
        auto f = random_state(3, 5000, rng);
        StateSet u = state_conservative(EosSpec(), 3, leaves_of(f));
        for (const Expr& e : {derived_c(u), derived_v_mag2(u), derived_p(u)}) {
            DenseVector want(Precision::f64, 5000), got(Precision::f64, 5000);
            evaluate(ref, e, want);
            dev::evaluate(be, e, got);
            if (!same_bits(want, got)) fail("derived quantity differs");
        }
        IdealGasEos gas;
        DenseVector want(Precision::f64, 5000), got(Precision::f64, 5000);
        evaluate(ref, gas.p_rhoe(leaf(f[0]), leaf(f[4])), want);
        dev::evaluate(be, gas.p_rhoe(leaf(f[0]), leaf(f[4])), got);
        if (!same_bits(want, got)) fail("eos p");
        // axpy-sin in place (dest aliases leaf y), as test_backend.cpp:37-48
        SplitMix64 r2(5);
        DenseVector x(Precision::f64, 777), y(Precision::f64, 777);
        for (std::size_t i = 0; i < 777; ++i) x.set(i, r2.uniform(0.25, 4.0));
        for (std::size_t i = 0; i < 777; ++i) y.set(i, r2.uniform(0.25, 4.0));
        DenseVector y_ref = y;
        evaluate(ref, constant(0.5, leaf(y_ref)) * elem_sin(leaf(x) + leaf(y_ref)), y_ref);
        dev::evaluate(be, constant(0.5, leaf(y)) * elem_sin(leaf(x) + leaf(y)), y);
        for (std::size_t i = 0; i < 777; ++i) {
            long long a, b;
            double va = y.at(i), vb = y_ref.at(i);
            std::memcpy(&a, &va, 8);
            std::memcpy(&b, &vb, 8);
            if (std::llabs(a - b) > 4) fail("axpy-sin beyond 4 ulp");
        }
        return "";
    });

    check("Jacobians + CFL on device vs the reference engine (d=3, f64 and f32)", [&] {
        for (Precision P : {Precision::f64, Precision::f32}) {
            SplitMix64 rng(21);
            auto f = random_state(3, 3001, rng, P);
            StateSet u = state_conservative(EosSpec(), 3, leaves_of(f));
            BlockExpr J = inviscid_flux_jacobian(u);
            BlockVectorGrid want(15, 5, P, 3001), got(15, 5, P, 3001);
            evaluate_block(ref, J, want);
            // the fused CFL reduction is a hand-written kernel; under
            // FVB_FORCE_LOWER the block itself runs lowered, without it
            const bool lowered = std::getenv("FVB_FORCE_LOWER") != nullptr;
            double lam = 0;
            if (lowered)
                dev::evaluate_block(be, J, got);
            else
                lam = dev::evaluate_block_cfl(be, J, got);
            for (std::size_t i = 0; i < 75; ++i)
                if (!same_bits(want.get(i), got.get(i))) fail("jacobian item " + std::to_string(i));
            if (lowered) continue;
            DenseVector ws(P, 3001);
            evaluate(ref, wave_speed(u), ws);
            double m = 0;
            for (std::size_t i = 0; i < 3001; ++i) m = std::fmax(m, ws.at(i));
            if (lam != m) fail("fused CFL max differs from the reference max");
            if (dev::reduce_max(be, wave_speed(u)) != m) fail("reduce_max differs");
        }
        return "";
    });

    check("host-side writes: constant items filled on the host, never over a plane the kernel reads", [&] {
        // Bare constant items of host destinations are filled by host threads
        // while the device pipeline streams the rest -- unless the
        // destination is also a leaf of the block (here item 0 reads the
        // plane item 1 overwrites with a constant: the reference reads the
        // old values, block.cpp:413-451) or another item's destination.
        const std::size_t n = 1'000'003;
        dev::DeviceBackend small = be;
        small.chunk_points = 1 << 16;  // many chunks: a racing fill would show
        for (Precision P : {Precision::f64, Precision::f32}) {
            SplitMix64 rng(5);
            DenseVector a = testutil::make_vec(P, n, rng);
            std::vector<DenseVector> w, g;
            for (int i = 0; i < 3; ++i) {
                w.emplace_back(P, n);
                g.emplace_back(P, n);
            }
            BlockColVector want(std::move(w)), got(std::move(g));
            for (BlockColVector* d : {&want, &got})
                for (std::size_t i = 0; i < n; ++i) d->get(1).set(i, double(i % 7) - 3.0);
            auto block = [&](BlockColVector& d) {
                const Expr b = leaf(d.get(1));
                return make_block_expr(3, 1, b * b + leaf(a), constant(2.5, b),
                                       constant(0.1, Precision::f32));
            };
            evaluate_block(ref, block(want), want);
            dev::evaluate_block(small, block(got), got);
            for (std::size_t r = 0; r < 3; ++r)
                if (!same_bits(want.get(r), got.get(r)))
                    fail("item " + std::to_string(r) + " differs from the reference");
        }
        return "";
    });

    check("narrowing rules on device: f32 constants, one rounding into a narrow store", [&] {
        // test_backend.cpp:122-138
        DenseVector ones(Precision::f32, 9000);
        for (std::size_t i = 0; i < 9000; ++i) ones.set(i, 1.0);
        DenseVector out(Precision::f32, 9000);
        dev::evaluate(be, leaf(ones) * constant(0.1, leaf(ones)), out);
        if (out.f32()[0] != 0.1f || static_cast<double>(out.f32()[8999]) == 0.1)
            fail("f32 constant not narrowed before use");
        SplitMix64 rng(81);
        DenseVector x = testutil::make_vec(Precision::f64, 9000, rng, 0.1, 0.9);
        DenseVector narrow(Precision::f32, 9000), want(Precision::f32, 9000);
        dev::evaluate(be, leaf(x) * leaf(x) + leaf(x), narrow);  // exact ops: bitwise
        evaluate(ref, leaf(x) * leaf(x) + leaf(x), want);
        if (!same_bits(narrow, want)) fail("wide result stored narrow differs");
        for (std::size_t i = 0; i < 9000; ++i)
            if (narrow.f32()[i] != static_cast<float>(x.at(i) * x.at(i) + x.at(i)))
                fail("not a single rounding");
        return "";
    });

    check("formulations agree on device: p, v^2 and the flux from either state", [&] {
        // test_fluid.cpp:213-232 and 331-345, at n = 20000, within 1e-12
        SplitMix64 rng(404);
        for (std::size_t d = 1; d <= 3; ++d) {
            const std::size_t n = 20000;
            auto f = random_state(d, n, rng);
            StateSet uc = state_conservative(EosSpec(), d, leaves_of(f));
            StateSet up = convert(uc, Formulation::Primitive);
            // the primitive state's fields on the device, then derived from them
            std::vector<DenseVector> pf;
            for (std::size_t i = 0; i < d + 2; ++i) pf.emplace_back(Precision::f64, n);
            BlockColVector pv(std::move(pf));
            dev::evaluate_block(be, up.block(), pv);
            std::vector<Expr> pl;
            for (std::size_t i = 0; i < d + 2; ++i) pl.push_back(leaf(pv.get(i)));
            StateSet upm = state_primitive(EosSpec(), d, pl);
            DenseVector pc(Precision::f64, n), pp(Precision::f64, n), vc(Precision::f64, n),
                vp(Precision::f64, n);
            dev::evaluate(be, derived_p(uc), pc);
            dev::evaluate(be, derived_p(upm), pp);
            dev::evaluate(be, derived_v_mag2(uc), vc);
            dev::evaluate(be, derived_v_mag2(upm), vp);
            for (std::size_t i = 0; i < n; ++i)
                if (!testutil::scalar_close(pc.at(i), pp.at(i), 1e-12) ||
                    !testutil::scalar_close(vc.at(i), vp.at(i), 1e-12))
                    fail("derived quantities disagree, d=" + std::to_string(d));
            BlockVectorGrid fc(d + 2, d, Precision::f64, n), fp(d + 2, d, Precision::f64, n);
            dev::evaluate_block(be, inviscid_flux(uc), fc);
            dev::evaluate_block(be, inviscid_flux(upm), fp);
            for (std::size_t k = 0; k < (d + 2) * d; ++k)
                for (std::size_t i = 0; i < n; ++i)
                    if (!testutil::scalar_close(fc.get(k).at(i), fp.get(k).at(i), 1e-12))
                        fail("primitive and conservative flux disagree, d=" + std::to_string(d));
        }
        return "";
    });

    check("a block wider than one launch (300 planes) runs as fused parts", [&] {
        SplitMix64 rng(71);
        const std::size_t n = 3001, items = 100;
        std::vector<DenseVector> in;
        for (std::size_t i = 0; i < 2 * items; ++i)
            in.push_back(testutil::make_vec(Precision::f64, n, rng));
        std::vector<BlockItem> bi;
        for (std::size_t i = 0; i < items; ++i)
            bi.push_back(BlockItem(leaf(in[2 * i]) * leaf(in[2 * i + 1]) - leaf(in[2 * i])));
        BlockExpr e(items, 1, bi);
        std::vector<DenseVector> wd, gd;
        for (std::size_t i = 0; i < items; ++i) {
            wd.emplace_back(Precision::f64, n);
            gd.emplace_back(Precision::f64, n);
        }
        BlockColVector want(std::move(wd)), got(std::move(gd));
        evaluate_block(ref, e, want);
        dev::evaluate_block(be, e, got);
        for (std::size_t i = 0; i < items; ++i)
            if (!same_bits(want.get(i), got.get(i))) fail("item " + std::to_string(i));
        return "";
    });

    check("column-major blocks and destination grids map items logically", [&] {
        // linear_index (block.hpp:14-18): a ColMajor grid stores item (r, c)
        // at c*nrow + r; items are still matched by (r, c)
        SplitMix64 rng(52);
        const std::size_t n = 9001;
        auto f = random_state(3, n, rng);
        StateSet u = state_conservative(EosSpec(), 3, leaves_of(f));
        BlockVectorGrid want(5, 3, Precision::f64, n, StorageOrder::ColMajor);
        BlockVectorGrid got(5, 3, Precision::f64, n, StorageOrder::ColMajor);
        evaluate_block(ref, inviscid_flux(u), want);
        dev::evaluate_block(be, inviscid_flux(u), got);
        for (std::size_t r = 0; r < 5; ++r)
            for (std::size_t c = 0; c < 3; ++c)
                if (!same_bits(want.item(r, c), got.item(r, c))) fail("flux into a ColMajor grid");
        // a ColMajor block expression of mixed items into a RowMajor grid
        DenseVector a = testutil::make_vec(Precision::f64, n, rng), b = testutil::make_vec(Precision::f64, n, rng);
        std::vector<BlockItem> items{BlockItem(leaf(a) * leaf(b)), BlockItem(elem_sqrt(leaf(a))),
                                     BlockItem(leaf(a) / leaf(b)), BlockItem(leaf(b) - leaf(a))};
        BlockExpr e(2, 2, items, StorageOrder::ColMajor);
        BlockVectorGrid w2(2, 2, Precision::f64, n), g2(2, 2, Precision::f64, n);
        evaluate_block(ref, e, w2);
        dev::evaluate_block(be, e, g2);
        for (std::size_t i = 0; i < 4; ++i)
            if (!same_bits(w2.get(i), g2.get(i))) fail("ColMajor block expression");
        return "";
    });

    check("asynchronous evaluations, Jacobian + device-side CFL max included, captured into a CUDA graph", [&] {
        // The reference's own calls -- evaluate_block of inviscid_flux and of
        // convert(.., Primitive) -- on resident leaves into tie'd device
        // planes, enqueued without host waits, captured once and replayed.
        SplitMix64 rng(61);
        const std::size_t n = 50001;
        auto f = random_state(3, n, rng);
        StateSet u = state_conservative(EosSpec(), 3, leaves_of(f));
        std::vector<dev::DeviceVector> dv;
        dev::Residency res;
        for (auto& v : f) {
            dv.emplace_back(v.precision(), v.size());
            dv.back().upload(v);
        }
        for (std::size_t i = 0; i < f.size(); ++i) res.bind(f[i], dv[i]);
        cudaStream_t s = nullptr;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) fail("stream");
        dev::DeviceBackend ab = be;
        ab.residency = &res;
        ab.stream = s;
        ab.synchronize = false;
        std::vector<dev::DeviceVector> fl, pr;
        for (int i = 0; i < 15; ++i) fl.emplace_back(Precision::f64, n);
        for (int i = 0; i < 5; ++i) pr.emplace_back(Precision::f64, n);
        dev::Tie tf, tp;
        for (auto& o : fl) tf.dests.push_back(&o);
        for (auto& o : pr) tp.dests.push_back(&o);
        BlockExpr flux = inviscid_flux(u);
        BlockExpr prim = convert(u, Formulation::Primitive).block();
        // the Jacobians + CFL step too, its maximum left on the device
        const bool lowered = std::getenv("FVB_FORCE_LOWER") != nullptr;
        BlockExpr J = inviscid_flux_jacobian(u);
        std::vector<dev::DeviceVector> jo;
        for (int i = 0; i < 75; ++i) jo.emplace_back(Precision::f64, n);
        dev::Tie tj;
        for (auto& o : jo) tj.dests.push_back(&o);
        dev::DeviceVector lam(Precision::f64, 1);
        dev::evaluate_block(ab, flux, tf);  // warm: keys resolved outside the capture
        dev::evaluate_block(ab, prim, tp);
        if (!lowered) dev::evaluate_block_cfl(ab, J, tj, lam);
        cudaStreamSynchronize(s);
        for (auto* v : {&fl, &pr, &jo})
            for (auto& o : *v) cudaMemsetAsync(o.data(), 0, o.byte_size(), s);
        cudaMemsetAsync(lam.data(), 0xff, 8, s);
        cudaStreamSynchronize(s);
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
            fail("begin capture");
        dev::evaluate_block(ab, flux, tf);
        dev::evaluate_block(ab, prim, tp);
        if (!lowered) dev::evaluate_block_cfl(ab, J, tj, lam);
        if (cudaStreamEndCapture(s, &g) != cudaSuccess) fail("end capture");
        std::size_t nodes = 0;
        cudaGraphGetNodes(g, nullptr, &nodes);
        if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) fail("instantiate");
        for (int rep = 0; rep < 3; ++rep) cudaGraphLaunch(ge, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) fail("graph replay");
        BlockVectorGrid want(5, 3, Precision::f64, n);
        evaluate_block(ref, flux, want);
        DenseVector tmp(Precision::f64, n);
        for (std::size_t i = 0; i < 15; ++i) {
            fl[i].download(tmp);
            if (!same_bits(tmp, want.get(i))) fail("graph flux item " + std::to_string(i));
        }
        StateSet w = convert(u, Formulation::Primitive);
        for (std::size_t i = 0; i < 5; ++i) {
            DenseVector wi(Precision::f64, n);
            evaluate(ref, w.field(i), wi);
            pr[i].download(tmp);
            if (!same_bits(tmp, wi)) fail("graph primitive field " + std::to_string(i));
        }
        if (!lowered) {
            BlockVectorGrid jw(15, 5, Precision::f64, n);
            evaluate_block(ref, J, jw);
            for (std::size_t i = 0; i < 75; ++i) {
                jo[i].download(tmp);
                if (!same_bits(tmp, jw.get(i))) fail("graph jacobian item " + std::to_string(i));
            }
            DenseVector ws(Precision::f64, n), lv(Precision::f64, 1);
            evaluate(ref, wave_speed(u), ws);
            double mx = 0;
            for (std::size_t i = 0; i < n; ++i) mx = std::fmax(mx, ws.at(i));
            lam.download(lv);
            if (lv.at(0) != mx) fail("graph CFL maximum differs");
        }
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        cudaStreamDestroy(s);
        return std::to_string(nodes) + " graph nodes";
    });

    check("host vectors over several devices (DeviceBackend::ordinals), flux + CFL", [&] {
        // Each ordinal streams its own slice; on this one-GPU box the same
        // device serves every slice, which exercises the slicing, the
        // per-slice pointer offsets and the exact max-combine.
        int devices = 0;
        cudaGetDeviceCount(&devices);
        for (std::size_t G : {2u, 3u}) {
            dev::DeviceBackend mb = be;
            for (std::size_t g = 0; g < G; ++g) mb.ordinals.push_back(int(g) % devices);
            SplitMix64 rng(40 + G);
            const std::size_t n = 100003;
            auto f = random_state(3, n, rng);
            StateSet u = state_conservative(EosSpec(), 3, leaves_of(f));
            BlockVectorGrid want(5, 3, Precision::f64, n), got(5, 3, Precision::f64, n);
            evaluate_block(ref, inviscid_flux(u), want);
            dev::evaluate_block(mb, inviscid_flux(u), got);
            for (std::size_t i = 0; i < 15; ++i)
                if (!same_bits(want.get(i), got.get(i))) fail("flux item " + std::to_string(i));
            const std::size_t m = 20011;
            auto g3 = random_state(3, m, rng, Precision::f32);
            StateSet w = state_conservative(EosSpec(), 3, leaves_of(g3));
            BlockExpr J = inviscid_flux_jacobian(w);
            BlockVectorGrid jw(15, 5, Precision::f32, m), jg(15, 5, Precision::f32, m);
            evaluate_block(ref, J, jw);
            // (the fused CFL reduction is a hand-written kernel: under
            // FVB_FORCE_LOWER the block runs lowered, without it)
            const bool lowered = std::getenv("FVB_FORCE_LOWER") != nullptr;
            const double lam = lowered ? 0.0 : dev::evaluate_block_cfl(mb, J, jg);
            if (lowered) dev::evaluate_block(mb, J, jg);
            for (std::size_t i = 0; i < 75; ++i)
                if (!same_bits(jw.get(i), jg.get(i))) fail("jacobian item " + std::to_string(i));
            if (lowered) continue;
            DenseVector ws(Precision::f32, m);
            evaluate(ref, wave_speed(w), ws);
            double mx = 0;
            for (std::size_t i = 0; i < m; ++i) mx = std::fmax(mx, ws.at(i));
            if (lam != mx) fail("sliced CFL max differs");
            if (dev::reduce_max(mb, wave_speed(w)) != mx) fail("sliced reduce_max differs");
        }
        return std::to_string(devices) + " visible device(s)";
    });

    check("device-resident leaves (Residency) and tie'd make_temp destinations", [&] {
        SplitMix64 rng(33);
        const std::size_t n = 100003;
        auto f = random_state(3, n, rng);
        StateSet u = state_conservative(EosSpec(), 3, leaves_of(f));
        std::vector<dev::DeviceVector> planes;
        dev::Residency res;
        for (auto& v : f) {
            planes.push_back(dev::make_temp(Precision::f64, n));
            planes.back().upload(v);
        }
        for (std::size_t i = 0; i < 5; ++i) res.bind(f[i], planes[i]);
        dev::DeviceBackend rb;
        rb.residency = &res;
        std::vector<dev::DeviceVector> out;
        for (int i = 0; i < 15; ++i) out.push_back(dev::make_temp(Precision::f64, n));
        dev::Tie t;
        for (auto& o : out) t.dests.push_back(&o);
        dev::evaluate_block(rb, inviscid_flux(u), t);
        BlockVectorGrid want(5, 3, Precision::f64, n);
        evaluate_block(ref, inviscid_flux(u), want);
        DenseVector tmp(Precision::f64, n);
        for (std::size_t i = 0; i < 15; ++i) {
            out[i].download(tmp);
            if (!same_bits(tmp, want.get(i))) fail("resident flux item " + std::to_string(i));
        }
        // tie() of cons->prim + c into three device temporaries, d=1
        auto g = random_state(1, n, rng);
        StateSet u1 = state_conservative(EosSpec(), 1, leaves_of(g));
        auto v = dev::make_temp(Precision::f64, n), p = dev::make_temp(Precision::f64, n),
             c = dev::make_temp(Precision::f64, n);
        BlockExpr vpc = make_block_expr(3, 1, convert(u1, Formulation::Primitive).field(1),
                                        derived_p(u1), derived_c(u1));
        dev::evaluate_block(be, vpc, dev::tie(v, p, c));
        DenseVector w(Precision::f64, n);
        evaluate(ref, derived_c(u1), w);
        c.download(tmp);
        if (!same_bits(tmp, w)) fail("tied sound speed");
        return "";
    });

    check("a reused block expression (launch-plan cache) follows new data, residency and vector changes", [&] {
        SplitMix64 rng(34);
        const std::size_t n = 4099;
        auto f = random_state(3, n, rng);
        StateSet u = state_conservative(EosSpec(), 3, leaves_of(f));
        const BlockExpr F = inviscid_flux(u);  // built once, evaluated many times
        std::vector<dev::DeviceVector> planes;
        dev::Residency res;
        for (auto& v : f) {
            planes.push_back(dev::make_temp(Precision::f64, n));
            planes.back().upload(v);
        }
        for (std::size_t i = 0; i < 5; ++i) res.bind(f[i], planes[i]);
        dev::DeviceBackend rb;
        rb.residency = &res;
        std::vector<dev::DeviceVector> out;
        for (int i = 0; i < 15; ++i) out.push_back(dev::make_temp(Precision::f64, n));
        dev::Tie t;
        for (auto& o : out) t.dests.push_back(&o);
        DenseVector tmp(Precision::f64, n);
        auto agree = [&](const char* what) {
            BlockVectorGrid want(5, 3, Precision::f64, n);
            evaluate_block(ref, F, want);
            for (std::size_t i = 0; i < 15; ++i) {
                out[i].download(tmp);
                if (!same_bits(tmp, want.get(i)))
                    fail(std::string(what) + ": item " + std::to_string(i));
            }
        };
        dev::evaluate_block(rb, F, t);
        dev::evaluate_block(rb, F, t);  // the cached plan
        agree("second call");
        // new state values (in place on host and device): the plan holds no data
        auto g = random_state(3, n, rng);
        for (std::size_t i = 0; i < 5; ++i) {
            std::memcpy(f[i].raw(), g[i].raw(), f[i].byte_size());
            planes[i].upload(f[i]);
        }
        dev::evaluate_block(rb, F, t);
        agree("new data");
        // unbind rhoE and change it on the host only: the evaluation must read
        // the host vector now, not the stale resident plane
        res.unbind(f[4]);
        const DenseVector saved = f[4];
        for (std::size_t i = 0; i < n; ++i) f[4].set(i, f[4].at(i) * 1.5);
        dev::evaluate_block(rb, F, t);
        agree("after unbind");
        res.bind(f[4], planes[4]);  // bound again: the (older) resident plane is read
        dev::evaluate_block(rb, F, t);
        std::memcpy(f[4].raw(), saved.raw(), f[4].byte_size());  // what the plane holds
        agree("after re-bind");
        // other destinations: a host grid, then another one
        BlockVectorGrid g1(5, 3, Precision::f64, n), g2(5, 3, Precision::f64, n), want(5, 3, Precision::f64, n);
        dev::evaluate_block(rb, F, g1);
        dev::evaluate_block(rb, F, g2);
        evaluate_block(ref, F, want);
        for (std::size_t i = 0; i < 15; ++i)
            if (!same_bits(g1.get(i), want.get(i)) || !same_bits(g2.get(i), want.get(i)))
                fail("host grids: item " + std::to_string(i));
        // single expressions reuse their plan the same way
        const Expr P = derived_p(u);
        DenseVector p1(Precision::f64, n), pw(Precision::f64, n);
        dev::evaluate(rb, P, p1);
        dev::evaluate(rb, P, p1);
        evaluate(ref, P, pw);
        if (!same_bits(p1, pw)) fail("cached evaluate");
        // a leaf reassigned to another length: refused, not served from the cache
        dev::DeviceBackend hb;  // no residency: host leaves
        dev::evaluate_block(hb, F, g1);
        dev::evaluate(hb, P, p1);
        f[2] = DenseVector(Precision::f64, n + 1);
        int refused = 0;
        try {
            dev::evaluate_block(hb, F, g1);
        } catch (const LengthMismatch&) {
            ++refused;
        }
        try {
            dev::evaluate(hb, P, p1);
        } catch (const LengthMismatch&) {
            ++refused;
        }
        if (refused != 2) fail("a resized leaf was not refused");
        return "";
    });

    check("aliased pass-through: flux into a grid whose row 0 is the momentum fields", [&] {
        // proj/src/block.cpp:419-422 skips an item whose destination is its
        // own bare leaf; the remaining items are still fused into one pass.
        SplitMix64 rng(0xA1);
        for (std::size_t d = 1; d <= 3; ++d) {
            const std::size_t n = 20000;
            auto f = random_state(d, n, rng);
            auto over = [&](BlockVectorGrid& g) {
                std::vector<Expr> lv{leaf(f[0])};
                for (std::size_t j = 0; j < d; ++j) {
                    g.item(0, j) = f[1 + j];
                    lv.push_back(leaf(g.item(0, j)));
                }
                lv.push_back(leaf(f[d + 1]));
                return state_conservative(EosSpec(), d, lv);
            };
            BlockVectorGrid want(d + 2, d, Precision::f64, n), got(d + 2, d, Precision::f64, n);
            StateSet uw = over(want), ug = over(got);
            evaluate_block(ref, inviscid_flux(uw), want);
            dev::evaluate_block(be, inviscid_flux(ug), got);
            for (std::size_t i = 0; i < (d + 2) * d; ++i)
                if (!same_bits(want.get(i), got.get(i)))
                    fail("d=" + std::to_string(d) + " item " + std::to_string(i));
        }
        return "";
    });

    check("in-place blocks keep the reference's item order (convert over its own state)", [&] {
        // Item 1 overwrites m with v; the pressure item after it then reads v
        // in the reference's item-by-item loop.  The device path detects the
        // hazard and evaluates item by item too.
        SplitMix64 rng(0xB2);
        std::size_t differs = 0;
        for (std::size_t d = 1; d <= 3; ++d) {
            const std::size_t n = 5000;
            auto f = random_state(d, n, rng);
            BlockColVector want{std::vector<DenseVector>(f)}, got{std::vector<DenseVector>(f)};
            auto over = [&](BlockColVector& v) {
                std::vector<Expr> lv;
                for (std::size_t i = 0; i < d + 2; ++i) lv.push_back(leaf(v.get(i)));
                return state_conservative(EosSpec(), d, lv);
            };
            StateSet uw = over(want), ug = over(got);
            evaluate_block(ref, convert(uw, Formulation::Primitive).block(), want);
            dev::evaluate_block(be, convert(ug, Formulation::Primitive).block(), got);
            for (std::size_t i = 0; i < d + 2; ++i)
                if (!same_bits(want.get(i), got.get(i)))
                    fail("d=" + std::to_string(d) + " field " + std::to_string(i));
            // the hazard is real: out of place, p differs
            StateSet u0 = state_conservative(EosSpec(), d, leaves_of(f));
            DenseVector p0(Precision::f64, n);
            StateSet w0 = convert(u0, Formulation::Primitive);
            evaluate(ref, w0.field(d + 1), p0);
            if (!same_bits(p0, want.get(d + 1))) ++differs;
        }
        if (differs != 3) fail("in-place and out-of-place results coincide");
        return "";
    });

    check("a later item overwriting a pass-through's source: convert with p written over rho", [&] {
        // convert(u, Primitive).block() = [rho, v.., p]: the fused kernel
        // covers the computed items and rho is a plain copy.  With p's
        // destination = the rho leaf itself, the reference copies rho at
        // item 0, before item d+1 overwrites it (block.cpp:413-451); the
        // copy must not run after the kernel.  Host leaves (staged path) and
        // resident leaves (device path, tie'd outputs) both.
        SplitMix64 rng(0xD4);
        for (std::size_t d = 1; d <= 3; ++d) {
            const std::size_t n = 5003;
            auto f = random_state(d, n, rng);
            // the grid's last item holds rho: p is written over its own leaf
            auto column = [&] {
                std::vector<DenseVector> c;
                for (std::size_t i = 0; i + 1 < d + 2; ++i) c.emplace_back(Precision::f64, n);
                c.push_back(f[0]);
                return BlockColVector(std::move(c));
            };
            auto state = [&](BlockColVector& col) {
                std::vector<Expr> lv{leaf(col.get(d + 1))};
                for (std::size_t i = 1; i < d + 2; ++i) lv.push_back(leaf(f[i]));
                return state_conservative(EosSpec(), d, lv);
            };
            BlockColVector want = column(), got = column();
            StateSet uw = state(want), ug = state(got);
            evaluate_block(ref, convert(uw, Formulation::Primitive).block(), want);
            dev::evaluate_block(be, convert(ug, Formulation::Primitive).block(), got);
            for (std::size_t i = 0; i < d + 2; ++i)
                if (!same_bits(want.get(i), got.get(i)))
                    fail("d=" + std::to_string(d) + " host item " + std::to_string(i));
            if (!same_bits(want.get(0), f[0])) fail("the reference's copy is not the old rho");
            // resident: every leaf bound, p tie'd over rho's resident plane
            BlockColVector rcol = column();
            StateSet ur = state(rcol);
            std::vector<dev::DeviceVector> planes;
            dev::Residency res;
            std::vector<const DenseVector*> hosts{&rcol.get(d + 1)};
            for (std::size_t i = 1; i < d + 2; ++i) hosts.push_back(&f[i]);
            for (const DenseVector* h : hosts) {
                planes.push_back(dev::make_temp(Precision::f64, n));
                planes.back().upload(*h);
            }
            for (std::size_t i = 0; i < hosts.size(); ++i) res.bind(*hosts[i], planes[i]);
            dev::DeviceBackend rb = be;
            rb.residency = &res;
            std::vector<dev::DeviceVector> outs;
            for (std::size_t i = 0; i + 1 < d + 2; ++i) outs.push_back(dev::make_temp(Precision::f64, n));
            dev::Tie t;
            for (auto& o : outs) t.dests.push_back(&o);
            t.dests.push_back(&planes[0]);
            dev::evaluate_block(rb, convert(ur, Formulation::Primitive).block(), t);
            DenseVector tmp(Precision::f64, n);
            for (std::size_t i = 0; i < d + 2; ++i) {
                (i + 1 < d + 2 ? outs[i] : planes[0]).download(tmp);
                if (!same_bits(want.get(i), tmp))
                    fail("d=" + std::to_string(d) + " resident item " + std::to_string(i));
            }
        }
        return "";
    });

    check("two items naming one destination: the later item's value stands", [&] {
        // tie(X, v.., X) for convert(u, Primitive).block(): item 0 copies rho
        // into X, item d+1 then writes p there (the reference's item order).
        SplitMix64 rng(0xD5);
        for (std::size_t d = 1; d <= 3; ++d) {
            const std::size_t n = 4099;
            auto f = random_state(d, n, rng);
            StateSet u = state_conservative(EosSpec(), d, leaves_of(f));
            std::vector<dev::DeviceVector> outs;
            for (std::size_t i = 0; i < d + 1; ++i) outs.push_back(dev::make_temp(Precision::f64, n));
            dev::Tie t;
            for (auto& o : outs) t.dests.push_back(&o);
            t.dests.push_back(&outs[0]);
            dev::evaluate_block(be, convert(u, Formulation::Primitive).block(), t);
            DenseVector want(Precision::f64, n), got(Precision::f64, n);
            evaluate(ref, derived_p(u), want);
            outs[0].download(got);
            if (!same_bits(want, got)) fail("d=" + std::to_string(d) + ": X is not p");
        }
        return "";
    });

    check("in place through a hand-written kernel: pressure into rhoE (d=3)", [&] {
        SplitMix64 rng(0xC3);
        const std::size_t n = 70000;
        auto f = random_state(3, n, rng);
        auto g = f;
        StateSet uf = state_conservative(EosSpec(), 3, leaves_of(f));
        StateSet ug = state_conservative(EosSpec(), 3, leaves_of(g));
        const std::string name =
            lookup_name(dev::structural_key(derived_p(ug), Precision::f64));
        evaluate(ref, derived_p(uf), f[4]);
        dev::evaluate(be, derived_p(ug), g[4]);
        if (!same_bits(f[4], g[4])) fail("in-place pressure differs");
        return "kernel " + name;
    });

    check("re-entrant: 4 host threads evaluate different blocks at once", [&] {
        // The reference's backends are stateless and re-entrant
        // (proj/src/backend_eval.cpp:280-346); the device path shares staging
        // buffers per device and must stay correct under concurrent callers.
        const std::size_t n = 300000;
        std::vector<std::string> errs(4);
        std::vector<std::thread> pool;
        for (int t = 0; t < 4; ++t)
            pool.emplace_back([&, t] {
                try {
                    SplitMix64 rng(0xD0 + t);
                    const std::size_t d = 1 + t % 3;
                    auto f = random_state(d, n, rng);
                    StateSet u = state_conservative(EosSpec(), d, leaves_of(f));
                    BlockVectorGrid want(d + 2, d, Precision::f64, n), got(d + 2, d, Precision::f64, n);
                    evaluate_block(Backend::scalar_ref(), inviscid_flux(u), want);
                    for (int rep = 0; rep < 3; ++rep) {
                        dev::evaluate_block(be, inviscid_flux(u), got);
                        for (std::size_t i = 0; i < (d + 2) * d; ++i)
                            if (!same_bits(want.get(i), got.get(i))) throw std::runtime_error("differs");
                    }
                } catch (const std::exception& e) {
                    errs[t] = e.what();
                }
            });
        for (auto& th : pool) th.join();
        for (int t = 0; t < 4; ++t)
            if (!errs[t].empty()) fail("thread " + std::to_string(t) + ": " + errs[t]);
        return "";
    });

    check("errors: unsupported expression, length/shape mismatch, tag conflict, empty tree", [&] {
        DenseVector a(Precision::f64, 10), b(Precision::f64, 11), out(Precision::f64, 10);
        bool threw = false;
        try {  // a non-finite constant: the reference's JIT refuses such trees too
            dev::evaluate(be, leaf(a) * constant(INFINITY, leaf(a)), out);
        } catch (const UnsupportedExpression&) {
            threw = true;
        }
        if (!threw) fail("non-finite constant did not throw UnsupportedExpression");
        threw = false;
        try {  // a bare sparse-matrix item has no vector value (block.cpp:427-428)
            SparseMatrix m(10, 10, {{0, 0, 1.0}});
            std::vector<DenseVector> col;
            col.emplace_back(Precision::f64, 10);
            BlockColVector y(std::move(col));
            dev::evaluate_block(be, make_block_expr(1, 1, m), y);
        } catch (const KindMismatch&) {
            threw = true;
        }
        if (!threw) fail("matrix item did not throw KindMismatch");
        threw = false;
        try {
            dev::evaluate(be, constant(0.5, leaf(a)) * elem_sin(leaf(a) + leaf(b)), out);
        } catch (const LengthMismatch&) {
            threw = true;
        }
        if (!threw) fail("no LengthMismatch");
        threw = false;
        try {
            SplitMix64 rng(1);
            auto f = random_state(3, 10, rng);
            StateSet u = state_conservative(EosSpec(), 3, leaves_of(f));
            BlockVectorGrid g(3, 3, Precision::f64, 10);
            dev::evaluate_block(be, inviscid_flux(u), g);
        } catch (const ShapeMismatch&) {
            threw = true;
        }
        if (!threw) fail("no ShapeMismatch");
        threw = false;
        try {  // validate(): one tag bound to two different leaves (backend_eval.cpp:245-250)
            DenseVector c(Precision::f64, 10);
            dev::evaluate(be, tag(1, leaf(a)) + tag(1, leaf(c)), out);
        } catch (const TagConflict&) {
            threw = true;
        }
        if (!threw) fail("no TagConflict");
        dev::evaluate(be, tag(1, leaf(a)) + tag(1, leaf(a)), out);  // same leaf: fine
        threw = false;
        try {
            dev::evaluate(be, Expr(), out);
        } catch (const Error&) {
            threw = true;
        }
        if (!threw) fail("empty expression did not throw");
        return "";
    });
}

}  // namespace

// The reference-facing plugin with host DenseVectors (pageable memory, as
// the reference allocates them) and with device-resident leaves: 3-D flux,
// fp64, timed with a host clock around whole evaluate_block calls.
void run_perf(std::size_t n) {
    dev::DeviceBackend be;
    SplitMix64 rng(0x5EED);
    auto f = random_state(3, n, rng);
    StateSet u = state_conservative(EosSpec(), 3, leaves_of(f));
    BlockVectorGrid grid(5, 3, Precision::f64, n);
    auto time = [&](const dev::DeviceBackend& b, const char* what) {
        dev::evaluate_block(b, inviscid_flux(u), grid);  // warm (allocations, key)
        const int reps = 3;
        auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < reps; ++r) dev::evaluate_block(b, inviscid_flux(u), grid);
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
        std::printf("{\"path\": \"%s\", \"points\": %zu, \"ms\": %.3f, \"gpts\": %.4f}\n", what, n,
                    s * 1e3, n / s / 1e9);
        std::fflush(stdout);
    };
    time(be, "evaluate_block, host DenseVectors (pageable) in and out");
    std::vector<dev::DeviceVector> dv;
    dev::Residency res;
    for (auto& v : f) {
        dv.emplace_back(v.precision(), v.size());
        dv.back().upload(v);
    }
    for (std::size_t i = 0; i < f.size(); ++i) res.bind(f[i], dv[i]);
    dev::DeviceBackend rb = be;
    rb.residency = &res;
    time(rb, "evaluate_block, resident leaves, host grid out");
    std::vector<dev::DeviceVector> outs;
    for (int i = 0; i < 15; ++i) outs.emplace_back(Precision::f64, n);
    dev::Tie tie;
    for (auto& o : outs) tie.dests.push_back(&o);
    dev::evaluate_block(rb, inviscid_flux(u), tie);
    const int reps = 10;
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) dev::evaluate_block(rb, inviscid_flux(u), tie);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
    std::printf("{\"path\": \"evaluate_block, resident leaves, tie'd device outputs\", \"points\": %zu, "
                "\"ms\": %.3f, \"gpts\": %.4f}\n", n, s * 1e3, n / s / 1e9);
    // the Jacobian block + CFL from and into host DenseVectors (pageable):
    // 30 constant entries filled and 18 duplicates copied host-side
    {
        const std::size_t nj = std::min<std::size_t>(n, 5'000'000);
        SplitMix64 rj(0x5EED);
        auto fj = random_state(3, nj, rj);
        StateSet uj = state_conservative(EosSpec(), 3, leaves_of(fj));
        BlockVectorGrid jg(15, 5, Precision::f64, nj);
        (void)dev::evaluate_block_cfl(be, inviscid_flux_jacobian(uj), jg);  // warm
        const int rj_reps = 3;
        auto tj0 = std::chrono::steady_clock::now();
        for (int r = 0; r < rj_reps; ++r) (void)dev::evaluate_block_cfl(be, inviscid_flux_jacobian(uj), jg);
        const double sj =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - tj0).count() / rj_reps;
        std::printf("{\"path\": \"evaluate_block_cfl(jacobian), host DenseVectors (pageable) in and out\", "
                    "\"points\": %zu, \"ms\": %.3f, \"gpts\": %.4f}\n", nj, sj * 1e3, nj / sj / 1e9);
    }
}

// Host overhead of one reference-API call at small n: the adapter's key
// building, lookup and launch, with resident leaves and tie'd outputs.
void run_overhead() {
    dev::DeviceBackend be;
    const std::size_t n = 1024;
    SplitMix64 rng(0x5EED);
    auto f = random_state(3, n, rng);
    StateSet u = state_conservative(EosSpec(), 3, leaves_of(f));
    std::vector<dev::DeviceVector> dv;
    dev::Residency res;
    for (auto& v : f) {
        dv.emplace_back(v.precision(), v.size());
        dv.back().upload(v);
    }
    for (std::size_t i = 0; i < f.size(); ++i) res.bind(f[i], dv[i]);
    be.residency = &res;
    std::vector<dev::DeviceVector> fo, jo;
    for (int i = 0; i < 15; ++i) fo.emplace_back(Precision::f64, n);
    for (int i = 0; i < 75; ++i) jo.emplace_back(Precision::f64, n);
    dev::Tie tf, tj;
    for (auto& o : fo) tf.dests.push_back(&o);
    for (auto& o : jo) tj.dests.push_back(&o);
    auto time = [&](const char* what, auto&& call) {
        for (int i = 0; i < 50; ++i) call();
        const int reps = 2000;
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < reps; ++i) call();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::printf("{\"call\": \"%s\", \"n\": %zu, \"us_per_call\": %.2f}\n", what, n,
                    s / reps * 1e6);
    };
    time("evaluate_block(inviscid_flux), resident, tie, synchronous", [&] {
        dev::evaluate_block(be, inviscid_flux(u), tf);
    });
    time("evaluate_block_cfl(jacobian), resident, tie", [&] {
        (void)dev::evaluate_block_cfl(be, inviscid_flux_jacobian(u), tj);
    });
    {
        // the same calls on expression objects built once (a time loop's
        // usual shape): the launch-plan cache serves every call after the first
        const BlockExpr F = inviscid_flux(u), J = inviscid_flux_jacobian(u);
        time("evaluate_block(inviscid_flux), reused tree, resident, tie, synchronous", [&] {
            dev::evaluate_block(be, F, tf);
        });
        time("evaluate_block_cfl(jacobian), reused tree, resident, tie", [&] {
            (void)dev::evaluate_block_cfl(be, J, tj);
        });
        std::vector<void*> in, fout;
        for (auto& d : dv) in.push_back(d.data());
        for (auto& o : fo) fout.push_back(o.data());
        time("fvb_flux direct C-ABI call + stream sync (the floor)", [&] {
            fvb_flux(nullptr, 3, 1, n, in.data(), fout.data(), nullptr);
            cudaStreamSynchronize(nullptr);
        });
    }
    volatile std::size_t sink = 0;
    time("build the tree inviscid_flux(u) only (reference code)", [&] {
        sink = sink + inviscid_flux(u).block_rows();
    });
    time("build the tree inviscid_flux_jacobian(u) only", [&] {
        sink = sink + inviscid_flux_jacobian(u).block_rows();
    });
    {
        BlockExpr J = inviscid_flux_jacobian(u);
        std::vector<Expr> items;
        for (std::size_t r = 0; r < J.block_rows(); ++r)
            for (std::size_t c = 0; c < J.block_cols(); ++c) items.push_back(J.item(r, c).as_expr());
        std::vector<Precision> dests(items.size(), Precision::f64);
        time("block_key of the Jacobian block only", [&] {
            sink = sink + dev::block_key(items, dests, 15, 5, nullptr).size();
        });
        const std::string key = dev::block_key(items, dests, 15, 5, nullptr);
        time("fvb_lookup of the Jacobian key only", [&] {
            fvb_kernel k;
            sink = sink + fvb_lookup(key.c_str(), &k);
        });
    }
    dev::DeviceBackend ab = be;
    ab.synchronize = false;
    time("evaluate_block(inviscid_flux), resident, tie, asynchronous", [&] {
        dev::evaluate_block(ab, inviscid_flux(u), tf);
    });
    cudaDeviceSynchronize();
    // one time step -- flux, conversion, Jacobians + CFL max on the device --
    // as reference-API calls, and the same step captured once as a CUDA graph
    cudaStream_t s = nullptr;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    ab.stream = s;
    std::vector<dev::DeviceVector> po;
    for (int i = 0; i < 5; ++i) po.emplace_back(Precision::f64, n);
    dev::Tie tp;
    for (auto& o : po) tp.dests.push_back(&o);
    dev::DeviceVector lam(Precision::f64, 1);
    BlockExpr F = inviscid_flux(u), P = convert(u, Formulation::Primitive).block(),
              J = inviscid_flux_jacobian(u);
    auto step = [&] {
        dev::evaluate_block(ab, F, tf);
        dev::evaluate_block(ab, P, tp);
        dev::evaluate_block_cfl(ab, J, tj, lam);
    };
    time("time step as 3 asynchronous reference-API calls (trees prebuilt)", [&] {
        step();
        cudaStreamSynchronize(s);
    });
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    step();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    time("the same time step replayed as one CUDA graph", [&] {
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
    });
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(s);
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "keys";
    if (mode == "overhead") {
        run_overhead();
        return 0;
    }
    if (mode == "perf") {
        run_perf(argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 20000000ull);
        return 0;
    }
    if (mode == "keys" || mode == "all") run_keys();
    if (mode == "gpu" || mode == "all") run_gpu();
    std::printf(failures ? "%d check(s) failed\n" : "all checks passed\n", failures);
    return failures ? 1 : 0;
}
