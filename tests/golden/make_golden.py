"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/libfvref.so, built by `make -C oracle` from
/root/reference) through its public API.

    python tests/golden/make_golden.py

Every array is the reference engine's own output (fvref::evaluate /
evaluate_block, scalar_ref backend), so the fixtures pin the oracle and the
device path to the reference bit for bit.  Inputs: the random_state of
proj/tests/acceptance.cpp:214-230 (seed 0x5eed), the worked state of
proj/tests/test_fluid.cpp:198-204/280-292, the EOS hand values of
test_fluid.cpp:92-106, the monatomic gas of test_fluid.cpp:347-353 and the
axpy-sin inputs of test_backend.cpp:23-35 (make_vec, seed 1).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

N = 37  # ragged on purpose: not a multiple of any vector width
DT = {"f64": np.float64, "f32": np.float32}


def main():
    R = oracle.reference()
    if R is None:
        raise SystemExit("build the reference first: make -C oracle")
    for prec in ("f64", "f32"):
        for d in (1, 2, 3):
            s = R.random_state(d, N, seed=0x5EED, prec=prec)
            # the worked state (d=3) / its 1-D analogue appended as the last point
            worked = {1: [2.0, 2.0, 14.0], 2: [2.0, 2.0, 4.0, 14.0], 3: [2.0, 2.0, 4.0, 4.0, 14.0]}[d]
            s = [np.append(a, DT[prec](w)) for a, w in zip(s, worked)]
            flux = R.flux(d, s)
            c2p = R.cons2prim(d, s)
            prim = [s[0]] + c2p[:d] + [c2p[d]]
            p2c = R.prim2cons(d, prim)
            vm = R.v_mag2(d, s)
            jac, lam = R.jacobian(d, s)
            ws, _ = R.wave_speed(d, s)
            np.savez(os.path.join(HERE, f"fluid_{prec}_d{d}.npz"), state=np.stack(s),
                     flux=np.stack(flux), cons2prim=np.stack(c2p), prim=np.stack(prim),
                     prim2cons=np.stack(p2c), v_mag2=vm, jacobian=np.stack(jac),
                     lambda_max=np.array(lam), wave_speed=ws)
    # axpy-sin: x = make_vec(seed 1) draws [0,n), y draws [n, 2n) (test_backend.cpp:25-27)
    n = 3000
    x = R.make_vec(1, 0, n)
    y = R.make_vec(1, n, n)
    np.savez(os.path.join(HERE, "axpy_sin.npz"), x=x, y=y, y_out=R.axpy_sin(x, y),
             x32=x.astype(np.float32), y32=y.astype(np.float32),
             y32_out=R.axpy_sin(x.astype(np.float32), y.astype(np.float32)))
    # EOS hand values and the monatomic closure
    rho = np.array([2.0, 1.5, 0.75])
    e = np.array([3.0, 2.0, 5.0])
    p, T = R.eos(rho, e)
    pm, Tm = R.eos(rho, e, cp=(5, 2), cv=(3, 2))
    mono = [np.array([1.0]), np.array([0.0]), np.array([3.0])]
    mono_c2p = R.cons2prim(1, mono, cp=(5, 2), cv=(3, 2))
    np.savez(os.path.join(HERE, "eos.npz"), rho=rho, e=e, p=p, T=T, p_mono=pm, T_mono=Tm,
             mono_state=np.stack(mono), mono_cons2prim=np.stack(mono_c2p))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
