"""The CPU oracle, pinned before it is trusted (CPU only).

Pins, in order of strength:
  1. bit-for-bit agreement with the UNMODIFIED reference built from
     /root/reference (oracle/_ref), on the reference's own random states;
  2. bit-for-bit agreement with the committed golden fixtures that
     tests/golden/make_golden.py generated from that reference build;
  3. the reference's own known-answer tests (test_fluid.cpp, acceptance.cpp),
     at the tolerances those tests state.
"""

import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
DT = {"f64": np.float64, "f32": np.float32}


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


def close(a, b, rtol):
    # scalar_close of proj/tests/oracle.hpp:97-102: rtol * max(|a|, |b|, 1)
    a, b = float(a), float(b)
    return abs(a - b) <= rtol * max(abs(a), abs(b), 1.0)


# ---- SplitMix64 -------------------------------------------------------------


def test_splitmix_random_access_matches_sequential(orc, ref):
    # rng.hpp:12-18 is sequential; the oracle and the device jump to draw k.
    seq = ref.make_vec(1, 0, 4000)
    assert bits_equal(orc.make_vec(1, 0, 4000), seq)
    assert bits_equal(orc.make_vec(1, 1234, 100), seq[1234:1334])


def test_splitmix_known_values(orc):
    # First outputs of SplitMix64 seeded with 0 (public test vector of the
    # generator rng.hpp implements).
    assert orc.draw(0, 0) == 0xE220A8397B1DCDAF
    assert orc.draw(0, 1) == 0x6E789E6AA1B965F4
    assert orc.draw(0, 2) == 0x06C45D188009454F


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_random_state_matches_reference(orc, ref, prec, dim):
    a = orc.random_state(dim, 777, seed=0x5EED, prec=prec)
    b = ref.random_state(dim, 777, seed=0x5EED, prec=prec)
    assert all(bits_equal(x, y) for x, y in zip(a, b))
    # random access: a slice of the global sequence equals the tail
    c = orc.random_state(dim, 100, seed=0x5EED, first=677, prec=prec)
    assert all(bits_equal(x, y[677:]) for x, y in zip(c, a))


# ---- bitwise against the reference build --------------------------------------


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [1, 2, 3])
@pytest.mark.parametrize("n", [0, 1, 7, 1025, 9000])
def test_fluid_blocks_bitwise_vs_reference(orc, ref, prec, dim, n):
    s = orc.random_state(dim, n, seed=0xF1 + n, prec=prec)
    for mine, theirs in [(orc.flux(dim, s), ref.flux(dim, s)),
                         (orc.cons2prim(dim, s), ref.cons2prim(dim, s)),
                         ([orc.v_mag2(dim, s)], [ref.v_mag2(dim, s)])]:
        assert len(mine) == len(theirs)
        assert all(bits_equal(x, y) for x, y in zip(mine, theirs))
    c = orc.cons2prim(dim, s)
    prim = [s[0]] + c[:dim] + [c[dim]]
    assert all(bits_equal(x, y) for x, y in zip(orc.prim2cons(dim, prim), ref.prim2cons(dim, prim)))
    assert all(bits_equal(x, y) for x, y in zip(orc.flux_prim(dim, prim), ref.flux_prim(dim, prim)))
    j, lam = orc.jacobian(dim, s)
    j2, lam2 = ref.jacobian(dim, s)
    assert all(bits_equal(x, y) for x, y in zip(j, j2))
    assert float(lam) == lam2


def test_parallel_reference_is_bitwise_scalar(ref):
    # The reference's own guarantee (bench.cpp:334-345) that the CPU baseline
    # we time in parallel computes the same bits as scalar_ref.
    s = ref.random_state(3, 20000, seed=7)
    a = ref.flux(3, s, workers=0)
    b = ref.flux(3, s, workers=4)
    assert all(bits_equal(x, y) for x, y in zip(a, b))


def test_gas_variants_bitwise_vs_reference(orc, ref):
    s = orc.random_state(2, 300, seed=99)
    g = orc.gas(cp=(5, 2), cv=(3, 2))
    mine = orc.flux(2, s, gas=g) + orc.cons2prim(2, s, gas=g) + orc.jacobian(2, s, gas=g)[0]
    theirs = (ref.flux(2, s, cp=(5, 2), cv=(3, 2)) + ref.cons2prim(2, s, cp=(5, 2), cv=(3, 2))
              + ref.jacobian(2, s, cp=(5, 2), cv=(3, 2))[0])
    assert all(bits_equal(x, y) for x, y in zip(mine, theirs))


def test_axpy_sin_bitwise_vs_reference(orc, ref):
    x = orc.make_vec(1, 0, 3000)
    y = orc.make_vec(1, 3000, 3000)
    assert bits_equal(orc.axpy_sin(x, y), ref.axpy_sin(x, y))
    assert bits_equal(orc.axpy_sin(x.astype(np.float32), y.astype(np.float32)),
                      ref.axpy_sin(x.astype(np.float32), y.astype(np.float32)))
    # compiled-JIT path (n >= 8192, backend_jit.cpp) in parallel as well
    x = orc.make_vec(5, 0, 20000)
    y = orc.make_vec(5, 20000, 20000)
    assert bits_equal(orc.axpy_sin(x, y), ref.axpy_sin(x, y, workers=3))


def test_eos_bitwise_vs_reference(orc, ref):
    rho = orc.make_vec(3, 0, 500, 0.5, 2.0)
    e = orc.make_vec(3, 500, 500, 0.5, 4.0)
    p, T = orc.eos(rho, e)
    p2, T2 = ref.eos(rho, e)
    assert bits_equal(p, p2) and bits_equal(T, T2)


# ---- golden fixtures (committed, generated from the reference) ---------------


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_oracle_reproduces_golden(orc, prec, dim):
    z = np.load(os.path.join(GOLDEN, f"fluid_{prec}_d{dim}.npz"))
    s = [np.ascontiguousarray(r) for r in z["state"]]
    assert bits_equal(np.stack(orc.flux(dim, s)), z["flux"])
    assert bits_equal(np.stack(orc.cons2prim(dim, s)), z["cons2prim"])
    prim = [np.ascontiguousarray(r) for r in z["prim"]]
    assert bits_equal(np.stack(orc.prim2cons(dim, prim)), z["prim2cons"])
    assert bits_equal(orc.v_mag2(dim, s), z["v_mag2"])
    j, lam = orc.jacobian(dim, s)
    assert bits_equal(np.stack(j), z["jacobian"])
    assert float(lam) == float(z["lambda_max"])
    assert float(orc.wave_speed_max(dim, s)) == float(z["lambda_max"])


def test_oracle_reproduces_golden_axpy(orc):
    z = np.load(os.path.join(GOLDEN, "axpy_sin.npz"))
    assert bits_equal(orc.make_vec(1, 0, 3000), z["x"])
    assert bits_equal(orc.make_vec(1, 3000, 3000), z["y"])
    assert bits_equal(orc.axpy_sin(z["x"], z["y"]), z["y_out"])
    assert bits_equal(orc.axpy_sin(z["x32"], z["y32"]), z["y32_out"])


def test_oracle_reproduces_golden_eos(orc):
    z = np.load(os.path.join(GOLDEN, "eos.npz"))
    p, T = orc.eos(z["rho"], z["e"])
    assert bits_equal(p, z["p"]) and bits_equal(T, z["T"])
    g = orc.gas(cp=(5, 2), cv=(3, 2))
    pm, Tm = orc.eos(z["rho"], z["e"], gas=g)
    assert bits_equal(pm, z["p_mono"]) and bits_equal(Tm, z["T_mono"])
    mono = [np.ascontiguousarray(r) for r in z["mono_state"]]
    assert bits_equal(np.stack(orc.cons2prim(1, mono, gas=g)), z["mono_cons2prim"])


# ---- the reference's own known answers --------------------------------------


def worked_state(prec="f64"):
    return [np.array([v], DT[prec]) for v in (2.0, 2.0, 4.0, 4.0, 14.0)]


def test_worked_flux_column(orc):
    # test_fluid.cpp:280-292 / acceptance.cpp:327-336: column 0 = [2,4,4,4,16]
    f = orc.flux(3, worked_state())
    col0 = [f[r * 3 + 0][0] for r in range(5)]
    assert col0 == [2.0, 4.0, 4.0, 4.0, 16.0]
    # columns 1 and 2 from the flux definition
    assert [f[r * 3 + 1][0] for r in range(5)] == [4.0, 4.0, 10.0, 8.0, 32.0]
    assert [f[r * 3 + 2][0] for r in range(5)] == [4.0, 4.0, 8.0, 10.0, 32.0]


def test_worked_pressure_and_vmag2(orc):
    # test_fluid.cpp:198-204: p = 2.0, v^2 = 9.0
    c = orc.cons2prim(3, worked_state())
    assert close(c[3][0], 2.0, 1e-14)
    assert close(orc.v_mag2(3, worked_state())[0], 9.0, 1e-14)
    # sound speed and wave speed, SURVEY A.5
    assert c[4][0] == 1.1832159566199232
    assert orc.wave_speed_max(3, worked_state()) == 4.183215956619923


def test_worked_jacobian(orc):
    # A_0 at the worked state, and A_k U = F_k (Euler homogeneity)
    j, lam = orc.jacobian(3, worked_state())
    A = np.array([x[0] for x in j]).reshape(3, 5, 5)
    want0 = [[0, 1, 0, 0, 0], [0.8, 1.6, -0.8, -0.8, 0.4], [-2, 2, 1, 0, 0], [-2, 2, 0, 1, 0],
             [-6.2, 7.6, -0.8, -0.8, 1.4]]
    assert np.allclose(A[0], want0, rtol=1e-14, atol=1e-14)
    U = np.array([2.0, 2.0, 4.0, 4.0, 14.0])
    f = orc.flux(3, worked_state())
    for k in range(3):
        Fk = np.array([f[r * 3 + k][0] for r in range(5)])
        assert np.allclose(A[k] @ U, Fk, rtol=1e-14, atol=1e-13)
    assert float(lam) == 4.183215956619923


def test_homogeneity_random_states(orc):
    # A_k(U) U = F_k(U) for every random state (ties the new Jacobian block
    # to the reference-pinned flux)
    for dim in (1, 2, 3):
        s = orc.random_state(dim, 200, seed=42)
        j, _ = orc.jacobian(dim, s)
        f = orc.flux(dim, s)
        w = dim + 2
        A = np.stack(j).reshape(dim, w, w, -1)
        U = np.stack(s)
        for k in range(dim):
            AU = np.einsum("rcn,cn->rn", A[k], U)
            Fk = np.stack([f[r * dim + k] for r in range(w)])
            assert np.allclose(AU, Fk, rtol=1e-12, atol=1e-12)


def test_eos_hand_values(orc):
    # test_fluid.cpp:92-106: rho=2, e=3 -> p=2.4, T=1.2
    p, T = orc.eos(np.array([2.0]), np.array([3.0]))
    assert close(p[0], 2.4, 1e-15) and close(T[0], 1.2, 1e-15)


def test_monatomic_pressure(orc):
    # test_fluid.cpp:347-353: cp=5/2, cv=3/2, rho=1, m=0, rhoE=3 -> p = 2.0
    g = orc.gas(cp=(5, 2), cv=(3, 2))
    c = orc.cons2prim(1, [np.array([1.0]), np.array([0.0]), np.array([3.0])], gas=g)
    assert close(c[1][0], 2.0, 1e-14)


def test_figure2_expression(orc):
    # test_expr.cpp:82-88: x=0, y=pi/2 -> 0.5*sin(x+y) = 0.5
    y = orc.axpy_sin(np.array([0.0]), np.array([math.pi / 2]))
    assert close(y[0], 0.5, 1e-15)


def test_1d_worked_cons2prim(orc):
    # rho=2, m=2, rhoE=14 -> u=1, p=5.2, c=1.9078784028338913
    c = orc.cons2prim(1, [np.array([2.0]), np.array([2.0]), np.array([14.0])])
    assert c[0][0] == 1.0 and close(c[1][0], 5.2, 1e-15) and c[2][0] == 1.9078784028338913


def test_thermodynamic_identities(orc):
    # acceptance.cpp:244-284: round trip and p = rho R T within 1e-12
    for dim in (1, 2, 3):
        s = orc.random_state(dim, 128, seed=0x7E6 + dim)
        c = orc.cons2prim(dim, s)
        prim = [s[0]] + c[:dim] + [c[dim]]
        back = orc.prim2cons(dim, prim)
        for a, b in zip(back, s[1:]):
            assert all(close(x, y, 1e-12) for x, y in zip(a, b))
        vm = orc.v_mag2(dim, s)
        e_int = (s[dim + 1] - 0.5 * (s[0] * vm)) / s[0]
        _, T = orc.eos(s[0], e_int)
        assert all(close(p, r * 1.0 * t, 1e-12) for p, r, t in zip(c[dim], s[0], T))


# ---- IEEE special values --------------------------------------------------------

SPECIAL = [0.0, -0.0, 1.0, -1.0, 5e-324, 1e300, float("inf"), float("-inf"), float("nan")]


def special_state(dim, prec="f64"):
    """Every combination of special values over (rho, m_0, rhoE), the other
    momenta 1.0: division by zero, overflow, NaN, denormals, negative rho."""
    import itertools
    pts = list(itertools.product(SPECIAL, SPECIAL, SPECIAL))
    rho = np.array([p[0] for p in pts])
    m0 = np.array([p[1] for p in pts])
    E = np.array([p[2] for p in pts])
    planes = [rho, m0] + [np.ones_like(rho)] * (dim - 1) + [E]
    return [np.ascontiguousarray(p.astype(DT[prec])) for p in planes]


def nan_aware_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    both_nan = np.isnan(a) & np.isnan(b)
    same = a.view(np.uint8).reshape(a.size, -1) == b.view(np.uint8).reshape(b.size, -1)
    return bool(np.all(both_nan | same.all(axis=1)))


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_special_values_vs_reference(orc, ref, prec, dim):
    # NaN payloads are platform-specific (x86 produces -nan); everything
    # else, including signed zeros, infinities and denormals, is bitwise.
    s = special_state(dim, prec)
    for mine, theirs in [(orc.flux(dim, s), ref.flux(dim, s)),
                         (orc.cons2prim(dim, s), ref.cons2prim(dim, s)),
                         (orc.jacobian(dim, s)[0], ref.jacobian(dim, s)[0])]:
        assert all(nan_aware_equal(x, y) for x, y in zip(mine, theirs))
    assert np.isnan(orc.wave_speed_max(dim, s)) and np.isnan(ref.jacobian(dim, s)[1])


# ---- CSR block matvec ------------------------------------------------


def random_csr(rng, rows, cols, max_row, empty_every=0):
    """Sorted, duplicate-free rows (as SparseMatrix stores them), some empty."""
    rp, ci, v = [0], [], []
    for r in range(rows):
        k = 0 if empty_every and r % empty_every == 0 else int(rng.integers(0, max_row + 1))
        c = np.sort(rng.choice(cols, min(k, cols), replace=False))
        ci += list(c)
        v += list(rng.uniform(-2.0, 2.0, len(c)))
        rp.append(len(ci))
    return (np.array(rp, np.uint64), np.array(ci, np.uint64), np.array(v, np.float64))


@pytest.mark.parametrize("y_prec", ["f64", "f32"])
@pytest.mark.parametrize("x_prec", ["f64", "f32"])
@pytest.mark.parametrize("m_prec", ["f64", "f32"])
def test_csr_matvec_matches_reference(orc, ref, y_prec, x_prec, m_prec):
    # The oracle's csr_matvec_acc restatement equals the reference's
    # block_matvec + evaluate_block bit for bit (block.cpp:345-356, 428-446):
    # short and long rows, empty rows, every precision combination.
    rng = np.random.default_rng(7)
    for rows, cols, max_row, empty in [(1, 1, 1, 0), (64, 50, 12, 5), (300, 1000, 200, 7),
                                       (2000, 2000, 7, 0)]:
        rp, ci, v = random_csr(rng, rows, cols, max_row, empty)
        x = rng.uniform(-2.0, 2.0, cols).astype(np.float64 if x_prec == "f64" else np.float32)
        want, stored = ref.csr_matvec(rp, ci, v, x, cols, y_prec=y_prec, m_prec=m_prec)
        y0 = np.zeros(rows, np.float64 if y_prec == "f64" else np.float32)
        got = orc.csr_matvec_acc(rp, ci, stored, x, y0)
        assert got.tobytes() == want.tobytes(), (rows, cols)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_eos_matches_reference(orc, ref, prec):
    # eos_ideal_p / eos_ideal_T (fluid.cpp:57-65) in both precisions, the
    # default and a monatomic gas, bit for bit against the reference build
    dt = np.float64 if prec == "f64" else np.float32
    rng = np.random.default_rng(4)
    rho = rng.uniform(0.1, 5.0, 10007).astype(dt)
    e = rng.uniform(0.1, 9.0, 10007).astype(dt)
    for cp, cv in [((7, 2), (5, 2)), ((5, 2), (3, 2))]:
        want_p, want_T = ref.eos(rho, e, cp=cp, cv=cv)
        got_p, got_T = orc.eos(rho, e, gas=orc.gas(cp, cv))
        assert got_p.tobytes() == want_p.tobytes() and got_T.tobytes() == want_T.tobytes()


# Gases with awkward rational constants: gamma - 1 = R/cv and gamma = cp/cv
# are then inexact doubles, so the narrowing and the operation order of
# every block are exercised (fluid.cpp:40-53).
RANDOM_GASES = [((7, 2), (5, 2)), ((5, 2), (3, 2)), ((9, 7), (1, 1)), ((13, 3), (11, 5)),
                ((100, 33), (2, 1)), ((31, 10), (7, 3))]


@pytest.mark.parametrize("cp,cv", RANDOM_GASES)
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_blocks_match_reference_for_many_gases(orc, ref, cp, cv, prec):
    g = orc.gas(cp=cp, cv=cv)
    for dim in (1, 3):
        s = orc.random_state(dim, 1031, seed=sum(cp) + 7 * sum(cv), prec=prec)
        mine = orc.flux(dim, s, gas=g) + orc.cons2prim(dim, s, gas=g)
        theirs = ref.flux(dim, s, cp=cp, cv=cv) + ref.cons2prim(dim, s, cp=cp, cv=cv)
        assert all(a.tobytes() == b.tobytes() for a, b in zip(mine, theirs)), (cp, cv, dim)
        jm, lm = orc.jacobian(dim, s, gas=g)
        jt, lt = ref.jacobian(dim, s, cp=cp, cv=cv)
        assert all(a.tobytes() == b.tobytes() for a, b in zip(jm, jt)) and lm == lt
