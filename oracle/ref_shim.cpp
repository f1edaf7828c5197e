// ref_shim.cpp -- C entry points into the UNMODIFIED fusevec reference.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference's own sources (/root/reference/proj/src/*.cpp, compiled in place,
// never copied) into oracle/_ref/libfvref.so.  The reference is built with
// -Dfusevec=fvref so its symbols live in namespace fvref:: and can never be
// confused with product code.  Used by tests/ (parity pinning of the C
// oracle, golden-fixture generation) and by bench.py --impl reference /
// cpu_baseline (the reference's own CPU path timed on the host cores).
//
// Every entry point drives the reference through its public API only:
// state_conservative / convert / derived_p / derived_v_mag2 / inviscid_flux
// (proj/include/fusevec/fluid.hpp), evaluate (backend.hpp:46) and
// evaluate_block (block.hpp:280-281).  The blocks the reference lacks
// (sound speed, Jacobians, wave speed) are composed
// from its public Expr API here and evaluated by the reference engine.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "fusevec/bench.hpp"
#include "fusevec/block.hpp"
#include "fusevec/fluid.hpp"
#include "fusevec/rng.hpp"

using namespace fvref;

namespace {

thread_local std::string g_err;

Precision prec_of(int p) { return p == 0 ? Precision::f32 : Precision::f64; }

Backend backend_of(int workers) {
    if (workers <= 0) return Backend::scalar_ref();
    return Backend::parallel(0, static_cast<std::size_t>(workers));
}

EosSpec gas_of(const long long* g) {
    if (!g) return EosSpec();
    return EosSpec(rational(g[0], g[1]), rational(g[2], g[3]));
}

DenseVector upload(Precision prec, std::size_t n, const void* src) {
    DenseVector v(prec, n);
    if (n) std::memcpy(v.raw(), src, v.byte_size());
    return v;
}

void download(const DenseVector& v, void* dst) {
    if (v.size()) std::memcpy(dst, v.raw(), v.byte_size());
}

std::vector<DenseVector> upload_planes(Precision prec, std::size_t n, std::size_t count,
                                       const void* const* in) {
    std::vector<DenseVector> out;
    out.reserve(count);
    for (std::size_t i = 0; i < count; ++i) out.push_back(upload(prec, n, in[i]));
    return out;
}

std::vector<Expr> leaves(const std::vector<DenseVector>& vs) {
    std::vector<Expr> out;
    for (const auto& v : vs) out.push_back(leaf(v));
    return out;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Sound speed A.2: elem_sqrt((constant(gamma, p) * p) / rho).
Expr sound_speed(const StateSet& u) {
    Expr p = derived_p(u);
    const Expr& rho = u.field(VarKind::Density);
    return elem_sqrt((constant(u.eos().gamma_value(), p) * p) / rho);
}

// Wave speed A.4: elem_sqrt(derived_v_mag2(u)) + c.
Expr wave_speed(const StateSet& u) { return elem_sqrt(derived_v_mag2(u)) + sound_speed(u); }

double gm1_of(const EosSpec& eos) { return (eos.R() / eos.cv()).value(); }

// Jacobian block A.3 composed from the public Expr API, [k][r][c] items of a
// (d*(d+2)) x (d+2) row-major BlockExpr.
BlockExpr jacobian_block(const StateSet& u) {
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
    auto c = [&](double x) { return constant(x, rho); };

    std::vector<BlockItem> items;
    items.reserve(d * w * w);
    for (std::size_t k = 0; k < d; ++k) {
        for (std::size_t col = 0; col < w; ++col) items.push_back(BlockItem(c(col == 1 + k ? 1.0 : 0.0)));
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
                items.push_back(BlockItem(acc.valid() ? acc : c(0.0)));
            }
            items.push_back(BlockItem(c(i == k ? gm1 : 0.0)));
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

double host_max(const DenseVector& lam) {
    // NaN-propagating max over lambda >= 0 (the CFL definition).
    double m = 0.0;
    for (std::size_t i = 0; i < lam.size(); ++i) {
        double x = lam.at(i);
        if (std::isnan(m)) break;
        if (std::isnan(x) || x > m) m = x;
    }
    return m;
}

using Clock = std::chrono::steady_clock;

template <class F>
double time_ns(F&& f) {
    auto t0 = Clock::now();
    f();
    return double(std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count());
}

// random_state of proj/tests/acceptance.cpp:214-230, sequential draws.
std::vector<DenseVector> random_state(std::size_t dim, std::size_t n, std::uint64_t seed,
                                      Precision prec) {
    SplitMix64 rng(seed);
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

}  // namespace

extern "C" {

const char* fvr_last_error() { return g_err.c_str(); }

unsigned fvr_hardware_threads() { return std::thread::hardware_concurrency(); }

// Sequential SplitMix64: n draws of uniform(lo, hi) starting at draw `first`.
int fvr_make_vec(std::uint64_t seed, std::uint64_t first, std::uint64_t n, double lo, double hi,
                 double* out) {
    return guarded([&] {
        SplitMix64 rng(seed);
        for (std::uint64_t k = 0; k < first; ++k) rng.next();
        for (std::uint64_t i = 0; i < n; ++i) out[i] = rng.uniform(lo, hi);
    });
}

int fvr_random_state(int dim, int prec, std::uint64_t seed, std::uint64_t n, void* const* out) {
    return guarded([&] {
        auto f = random_state(std::size_t(dim), n, seed, prec_of(prec));
        for (std::size_t i = 0; i < f.size(); ++i) download(f[i], out[i]);
    });
}

int fvr_axpy_sin(int prec, std::uint64_t n, const void* x, void* y, int workers) {
    return guarded([&] {
        DenseVector X = upload(prec_of(prec), n, x), Y = upload(prec_of(prec), n, y);
        Expr e = constant(0.5, leaf(Y)) * elem_sin(leaf(X) + leaf(Y));
        evaluate(backend_of(workers), e, Y);  // aliased, as test_backend.cpp:37-48
        download(Y, y);
    });
}

int fvr_flux(const long long* gas, int dim, int prec, std::uint64_t n, const void* const* in,
             void* const* out, int workers) {
    return guarded([&] {
        auto f = upload_planes(prec_of(prec), n, std::size_t(dim) + 2, in);
        StateSet u = state_conservative(gas_of(gas), std::size_t(dim), leaves(f));
        BlockVectorGrid grid(std::size_t(dim) + 2, std::size_t(dim), prec_of(prec), n);
        evaluate_block(backend_of(workers), inviscid_flux(u), grid);
        for (std::size_t i = 0; i < std::size_t(dim + 2) * std::size_t(dim); ++i)
            download(grid.get(i), out[i]);
    });
}

int fvr_flux_prim(const long long* gas, int dim, int prec, std::uint64_t n,
                  const void* const* in, void* const* out, int workers) {
    return guarded([&] {
        auto f = upload_planes(prec_of(prec), n, std::size_t(dim) + 2, in);
        StateSet w = state_primitive(gas_of(gas), std::size_t(dim), leaves(f));
        BlockVectorGrid grid(std::size_t(dim) + 2, std::size_t(dim), prec_of(prec), n);
        evaluate_block(backend_of(workers), inviscid_flux(w), grid);
        for (std::size_t i = 0; i < std::size_t(dim + 2) * std::size_t(dim); ++i)
            download(grid.get(i), out[i]);
    });
}

int fvr_cons2prim(const long long* gas, int dim, int prec, std::uint64_t n,
                  const void* const* in, void* const* out, int workers) {
    return guarded([&] {
        auto f = upload_planes(prec_of(prec), n, std::size_t(dim) + 2, in);
        StateSet u = state_conservative(gas_of(gas), std::size_t(dim), leaves(f));
        StateSet w = convert(u, Formulation::Primitive);
        Backend be = backend_of(workers);
        DenseVector tmp(prec_of(prec), n);
        for (int j = 0; j < dim + 1; ++j) {
            evaluate(be, w.field(std::size_t(j) + 1), tmp);
            download(tmp, out[j]);
        }
        evaluate(be, sound_speed(u), tmp);
        download(tmp, out[dim + 1]);
    });
}

int fvr_prim2cons(const long long* gas, int dim, int prec, std::uint64_t n,
                  const void* const* in, void* const* out, int workers) {
    return guarded([&] {
        auto f = upload_planes(prec_of(prec), n, std::size_t(dim) + 2, in);
        StateSet w = state_primitive(gas_of(gas), std::size_t(dim), leaves(f));
        StateSet u = convert(w, Formulation::Conservative);
        DenseVector tmp(prec_of(prec), n);
        for (int j = 0; j < dim + 1; ++j) {
            evaluate(backend_of(workers), u.field(std::size_t(j) + 1), tmp);
            download(tmp, out[j]);
        }
    });
}

int fvr_v_mag2(int dim, int prec, std::uint64_t n, const void* const* in, void* out,
               int workers) {
    return guarded([&] {
        auto f = upload_planes(prec_of(prec), n, std::size_t(dim) + 2, in);
        StateSet u = state_conservative(EosSpec(), std::size_t(dim), leaves(f));
        DenseVector tmp(prec_of(prec), n);
        evaluate(backend_of(workers), derived_v_mag2(u), tmp);
        download(tmp, out);
    });
}

int fvr_eos(const long long* gas, int prec, std::uint64_t n, const void* rho, const void* e,
            void* p_out, void* T_out) {
    return guarded([&] {
        DenseVector R = upload(prec_of(prec), n, rho), E = upload(prec_of(prec), n, e);
        IdealGasEos g(gas_of(gas));
        DenseVector tmp(prec_of(prec), n);
        evaluate(Backend::scalar_ref(), g.p_rhoe(leaf(R), leaf(E)), tmp);
        download(tmp, p_out);
        evaluate(Backend::scalar_ref(), g.T_rhoe(leaf(R), leaf(E)), tmp);
        download(tmp, T_out);
    });
}

int fvr_jacobian(const long long* gas, int dim, int prec, std::uint64_t n,
                 const void* const* in, void* const* out, double* lambda_max, int workers) {
    return guarded([&] {
        auto f = upload_planes(prec_of(prec), n, std::size_t(dim) + 2, in);
        StateSet u = state_conservative(gas_of(gas), std::size_t(dim), leaves(f));
        BlockExpr J = jacobian_block(u);
        const std::size_t w = std::size_t(dim) + 2;
        BlockVectorGrid grid(std::size_t(dim) * w, w, prec_of(prec), n);
        Backend be = backend_of(workers);
        evaluate_block(be, J, grid);
        for (std::size_t i = 0; i < std::size_t(dim) * w * w; ++i) download(grid.get(i), out[i]);
        if (lambda_max) {
            DenseVector lam(prec_of(prec), n);
            evaluate(be, wave_speed(u), lam);
            *lambda_max = host_max(lam);
        }
    });
}

int fvr_wave_speed(const long long* gas, int dim, int prec, std::uint64_t n,
                   const void* const* in, void* out, double* lambda_max, int workers) {
    return guarded([&] {
        auto f = upload_planes(prec_of(prec), n, std::size_t(dim) + 2, in);
        StateSet u = state_conservative(gas_of(gas), std::size_t(dim), leaves(f));
        DenseVector lam(prec_of(prec), n);
        evaluate(backend_of(workers), wave_speed(u), lam);
        if (out) download(lam, out);
        if (lambda_max) *lambda_max = host_max(lam);
    });
}

// ---------------------------------------------------------------------------
// CPU baseline timing: the reference's own path, inputs resident in host
// memory before the clock starts, one JIT warm-up, median over `reps`
// (the reference's method: proj/src/bench.cpp:17-51).  `which`:
//   0 = 3D-style flux evaluate_block(inviscid_flux(u))         (C3/C5)
//   1 = cons->prim fields + sound speed, one evaluate per field (C2)
//   2 = Jacobian evaluate_block + evaluate(lambda) + host max   (C4)
//   3 = axpy-sin y = 0.5*sin(x+y), in place                     (C1)
//   4 = derived_v_mag2 (the paper's micro-benchmark)
//   5 = prim->cons fields, 6 = primitive-formulation flux,
//   7 = EOS p and T, 8 = standalone CFL lambda + host max
// Writes per-rep nanoseconds into times_ns[0..reps).
// ---------------------------------------------------------------------------
int fvr_time_config(int which, int dim, int prec, std::uint64_t n, int workers, int reps,
                    std::uint64_t seed, double* times_ns) {
    return guarded([&] {
        const Precision P = prec_of(prec);
        Backend be = backend_of(workers);
        std::vector<double> t;
        if (which == 3) {
            SplitMix64 rng(seed);
            DenseVector x(P, n), y(P, n);
            for (std::size_t i = 0; i < n; ++i) x.set(i, rng.uniform(0.25, 4.0));
            for (std::size_t i = 0; i < n; ++i) y.set(i, rng.uniform(0.25, 4.0));
            Expr e = constant(0.5, leaf(y)) * elem_sin(leaf(x) + leaf(y));
            evaluate(be, e, y);
            for (int r = 0; r < reps; ++r) times_ns[r] = time_ns([&] { evaluate(be, e, y); });
            return;
        }
        auto f = random_state(std::size_t(dim), n, seed, P);
        StateSet u = state_conservative(EosSpec(), std::size_t(dim), leaves(f));
        const std::size_t d = std::size_t(dim), w = d + 2;
        if (which == 0) {
            BlockExpr flux = inviscid_flux(u);
            BlockVectorGrid grid(w, d, P, n);
            evaluate_block(be, flux, grid);
            for (int r = 0; r < reps; ++r)
                times_ns[r] = time_ns([&] { evaluate_block(be, flux, grid); });
        } else if (which == 1) {
            StateSet prim = convert(u, Formulation::Primitive);
            Expr c = sound_speed(u);
            std::vector<DenseVector> out(d + 2, DenseVector(P, n));
            auto run = [&] {
                for (std::size_t j = 0; j < d + 1; ++j) evaluate(be, prim.field(j + 1), out[j]);
                evaluate(be, c, out[d + 1]);
            };
            run();
            for (int r = 0; r < reps; ++r) times_ns[r] = time_ns(run);
        } else if (which == 2) {
            BlockExpr J = jacobian_block(u);
            Expr lam_e = wave_speed(u);
            BlockVectorGrid grid(d * w, w, P, n);
            DenseVector lam(P, n);
            volatile double sink = 0;
            auto run = [&] {
                evaluate_block(be, J, grid);
                evaluate(be, lam_e, lam);
                sink = host_max(lam);
            };
            run();
            for (int r = 0; r < reps; ++r) times_ns[r] = time_ns(run);
            (void)sink;
        } else if (which == 4) {
            // the paper's micro-benchmark: derived_v_mag2 (bench.cpp:153-206)
            Expr vm = derived_v_mag2(u);
            DenseVector out(P, n);
            evaluate(be, vm, out);
            for (int r = 0; r < reps; ++r) times_ns[r] = time_ns([&] { evaluate(be, vm, out); });
        } else if (which == 5 || which == 6) {
            // the same planes read as a primitive state [rho, v..., p]:
            // 5 = convert(prim, Conservative), one evaluate per computed field
            // 6 = the primitive-formulation flux (fluid.cpp:290-298)
            StateSet pr = state_primitive(EosSpec(), d, leaves(f));
            if (which == 5) {
                StateSet cons = convert(pr, Formulation::Conservative);
                std::vector<DenseVector> out(d + 1, DenseVector(P, n));
                auto run = [&] {
                    for (std::size_t j = 0; j < d + 1; ++j) evaluate(be, cons.field(j + 1), out[j]);
                };
                run();
                for (int r = 0; r < reps; ++r) times_ns[r] = time_ns(run);
            } else {
                BlockExpr flux = inviscid_flux(pr);
                BlockVectorGrid grid(w, d, P, n);
                evaluate_block(be, flux, grid);
                for (int r = 0; r < reps; ++r)
                    times_ns[r] = time_ns([&] { evaluate_block(be, flux, grid); });
            }
        } else if (which == 7) {
            // the ideal-gas EOS closures p(rho, e) and T(rho, e) (fluid.cpp:57-65)
            const Expr rho = leaf(f[0]), e = leaf(f[d + 1]);
            Expr pe = eos_ideal_p(rho, e, EosSpec()), te = eos_ideal_T(rho, e, EosSpec());
            DenseVector p(P, n), T(P, n);
            auto run = [&] {
                evaluate(be, pe, p);
                evaluate(be, te, T);
            };
            run();
            for (int r = 0; r < reps; ++r) times_ns[r] = time_ns(run);
        } else if (which == 8) {
            // standalone CFL: evaluate(lambda) + host max
            Expr lam_e = wave_speed(u);
            DenseVector lam(P, n);
            volatile double sink = 0;
            auto run = [&] {
                evaluate(be, lam_e, lam);
                sink = host_max(lam);
            };
            run();
            for (int r = 0; r < reps; ++r) times_ns[r] = time_ns(run);
            (void)sink;
        } else {
            throw Error("unknown timing config");
        }
    });
}

// y = A x through the reference's block layer: a 1x1 BlockMatrixView of the
// CSR matrix (rows given as sorted, duplicate-free triplets, which the
// SparseMatrix constructor stores unchanged: block.cpp:15-48) applied with
// block_matvec and evaluate_block (block.cpp:264-298, 428-446), i.e.
// y[r] = 0 + csr_matvec_acc row r.  v_stored receives the stored values
// (narrowed to prec_m, block.cpp:45) when not NULL.
int fvr_csr_matvec(int prec_y, int prec_x, int prec_m, std::uint64_t rows, std::uint64_t cols,
                   const std::uint64_t* rp, const std::uint64_t* ci, const double* v,
                   const void* x, void* y, double* v_stored) {
    return guarded([&] {
        std::vector<Triplet> trips;
        trips.reserve(rows ? rp[rows] : 0);
        for (std::uint64_t r = 0; r < rows; ++r)
            for (std::uint64_t k = rp[r]; k < rp[r + 1]; ++k)
                trips.push_back({std::size_t(r), std::size_t(ci[k]), v[k]});
        SparseMatrix a(rows, cols, trips, prec_of(prec_m));
        if (v_stored && !a.values().empty())
            std::memcpy(v_stored, a.values().data(), a.values().size() * sizeof(double));
        DenseVector xv = upload(prec_of(prec_x), cols, x);
        std::vector<DenseVector> yv;
        yv.emplace_back(prec_of(prec_y), rows);
        BlockColVector out(std::move(yv));
        BlockMatrixView view(1, 1, {&a});
        evaluate_block(Backend::scalar_ref(), block_matvec(view, BlockExpr(1, 1, {BlockItem(xv)})),
                       out);
        download(out.get(0), y);
    });
}

// The 7-point Laplacian on an n^3 grid (the PDE stencil the block layer's
// matvec serves), y = A x timed through evaluate_block as above.  The
// reference's csr_matvec_acc is serial whatever the backend.
int fvr_time_csr(std::uint64_t n, int reps, double* times_ns, std::uint64_t* nnz_out) {
    return guarded([&] {
        const std::uint64_t rows = n * n * n;
        std::vector<Triplet> trips;
        trips.reserve(rows * 7);
        const long long off[7] = {-(long long)(n * n), -(long long)n, -1, 0, 1, (long long)n,
                                  (long long)(n * n)};
        for (std::uint64_t r = 0; r < rows; ++r) {
            const std::uint64_t i = r % n, j = (r / n) % n, k = r / (n * n);
            const bool ok[7] = {k > 0, j > 0, i > 0, true, i + 1 < n, j + 1 < n, k + 1 < n};
            for (int t = 0; t < 7; ++t)
                if (ok[t]) trips.push_back({std::size_t(r), std::size_t((long long)r + off[t]),
                                            t == 3 ? 6.0 : -1.0});
        }
        SparseMatrix a(rows, rows, trips);
        *nnz_out = a.nnz();
        SplitMix64 rng(7);
        DenseVector xv(Precision::f64, rows);
        for (std::uint64_t i = 0; i < rows; ++i) xv.set(i, rng.uniform(-1.0, 1.0));
        std::vector<DenseVector> yv;
        yv.emplace_back(Precision::f64, rows);
        BlockColVector out(std::move(yv));
        BlockMatrixView view(1, 1, {&a});
        BlockExpr e = block_matvec(view, BlockExpr(1, 1, {BlockItem(xv)}));
        evaluate_block(Backend::scalar_ref(), e, out);
        for (int r = 0; r < reps; ++r)
            times_ns[r] = time_ns([&] { evaluate_block(Backend::scalar_ref(), e, out); });
    });
}

// The reference's own benchmark record (run_miniapp, proj/src/bench.cpp:294-384).
int fvr_run_miniapp(int prec, std::uint64_t n, int workers, double* median_ns,
                    double* overhead_ratio) {
    return guarded([&] {
        BenchConfig cfg;
        cfg.suite = "miniapp";
        cfg.sizes = {std::size_t(n)};
        cfg.precision = prec_of(prec);
        cfg.backend = workers > 0 ? BackendKind::Parallel : BackendKind::ScalarRef;
        cfg.workers = unsigned(std::max(workers, 0));
        auto recs = run_miniapp(cfg);
        *median_ns = recs.at(0).median_ns;
        *overhead_ratio = recs.at(0).overhead_ratio;
    });
}

}  // extern "C"
