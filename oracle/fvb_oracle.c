/*
 * fvb_oracle.c -- CPU oracle for the fused compressible-flow evaluation path.
 *
 * TEST INFRASTRUCTURE ONLY (see fvb_oracle.h for the contract and how it is
 * pinned).  Build with -ffp-contract=off (oracle/Makefile), matching the
 * reference's own flag (proj/CMakeLists.txt:11-14).
 */
#include "fvb_oracle.h"

#include <math.h>

fvo_gas fvo_default_gas(void) {
    /* EosSpec() = cp 7/2, cv 5/2 (proj/include/fusevec/fluid.hpp:31):
     * gamma = 7/5, R = 1, gm1 = R/cv = 2/5 (proj/src/fluid.cpp:53). */
    fvo_gas g;
    g.gm1 = 2.0 / 5.0;
    g.gamma = 7.0 / 5.0;
    g.cv = 5.0 / 2.0;
    return g;
}

uint64_t fvo_splitmix64_draw(uint64_t seed, uint64_t k) {
    /* proj/include/fusevec/rng.hpp:12-18 */
    uint64_t z = seed + (k + 1u) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

double fvo_uniform(uint64_t seed, uint64_t k, double lo, double hi) {
    /* proj/include/fusevec/rng.hpp:21-23 */
    double u = (double)(fvo_splitmix64_draw(seed, k) >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
}

#define FVO_T double
#define FVO_SFX f64
#define FVO_SIN sin
#define FVO_SQRT sqrt
#include "fvb_oracle_body.inc"
#undef FVO_T
#undef FVO_SFX
#undef FVO_SIN
#undef FVO_SQRT

#define FVO_T float
#define FVO_SFX f32
#define FVO_SIN sinf
#define FVO_SQRT sqrtf
#include "fvb_oracle_body.inc"
#undef FVO_T
#undef FVO_SFX
#undef FVO_SIN
#undef FVO_SQRT

void fvo_eos_p_f64(fvo_gas g, uint64_t n, const double* rho, const double* e, double* p) {
    /* eos_ideal_p: rho_e = rho*e; constant(gm1, rho_e) * rho_e
     * (proj/src/fluid.cpp:57-60). */
    for (uint64_t i = 0; i < n; ++i) p[i] = g.gm1 * (rho[i] * e[i]);
}

void fvo_eos_T_f64(fvo_gas g, uint64_t n, const double* e, double* T) {
    /* eos_ideal_T: e / constant(cv, e) (proj/src/fluid.cpp:62-65). */
    for (uint64_t i = 0; i < n; ++i) T[i] = e[i] / g.cv;
}

void fvo_eos_p_f32(fvo_gas g, uint64_t n, const float* rho, const float* e, float* p) {
    const float gm1 = (float)g.gm1;
    for (uint64_t i = 0; i < n; ++i) p[i] = gm1 * (rho[i] * e[i]);
}

void fvo_eos_T_f32(fvo_gas g, uint64_t n, const float* e, float* T) {
    const float cv = (float)g.cv;
    for (uint64_t i = 0; i < n; ++i) T[i] = e[i] / cv;
}

void fvo_wave_speed_f64(fvo_gas g, int dim, uint64_t n, const double* const* in, double* out) {
    for (uint64_t i = 0; i < n; ++i) {
        double rho, m[3], rho_E;
        load_state_f64(dim, in, i, &rho, m, &rho_E);
        out[i] = lambda_at_f64(g.gm1, g.gamma, dim, rho, m, rho_E);
    }
}

/* csr_matvec_acc_t<TY, TX> (proj/src/block.cpp:345-356). */
#define FVO_CSR(NAME, TY, TX)                                                          \
    void NAME(uint64_t rows, const uint64_t* rp, const uint64_t* ci, const double* v,   \
              const TX* x, TY* y) {                                                    \
        for (uint64_t r = 0; r < rows; ++r) {                                          \
            TY acc = 0;                                                                \
            for (uint64_t k = rp[r]; k < rp[r + 1]; ++k)                               \
                acc += (TY)v[k] * (TY)x[ci[k]];                                        \
            y[r] += acc;                                                               \
        }                                                                              \
    }
FVO_CSR(fvo_csr_matvec_acc_yd_xd, double, double)
FVO_CSR(fvo_csr_matvec_acc_yd_xs, double, float)
FVO_CSR(fvo_csr_matvec_acc_ys_xd, float, double)
FVO_CSR(fvo_csr_matvec_acc_ys_xs, float, float)
#undef FVO_CSR
