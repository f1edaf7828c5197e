"""CPU oracle for the fused compressible-flow path -- TEST INFRASTRUCTURE ONLY.

Two checkers, both plain CPU code, loaded with ctypes over numpy arrays:

* ``Oracle`` -- ``build/libfvb_oracle.so``: the C restatement of the
  reference's per-element arithmetic (fvb_oracle.c, every function citing the
  reference file:line it follows).
* ``Reference`` -- ``_ref/libfvref.so``: the UNMODIFIED fusevec reference,
  compiled from /root/reference by oracle/Makefile (namespace fvref), driven
  through its public API by ref_shim.cpp.  Present wherever it was built
  (here, and on the GPU box via the gpurun snapshot); ``reference()`` returns
  None when the file is absent.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package, and only as the checker / reported baseline.  The
product (libfvb.so and paper_1809_09851_b200) never touches it.
"""

from __future__ import annotations

import ctypes
import os
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libfvb_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfvref.so")

_DT = {"f64": np.float64, "f32": np.float32}
_PREC = {"f32": 0, "f64": 1}


def _prec_of(arr) -> str:
    return "f64" if arr.dtype == np.float64 else "f32"


def _pp(arrs):
    out = (ctypes.c_void_p * max(len(arrs), 1))()
    for i, a in enumerate(arrs):
        assert a.flags["C_CONTIGUOUS"]
        out[i] = a.ctypes.data
    return out


class GasC(ctypes.Structure):
    _fields_ = [("gm1", ctypes.c_double), ("gamma", ctypes.c_double), ("cv", ctypes.c_double)]


def gas_constants(cp=(7, 2), cv=(5, 2)):
    """(gm1, gamma, cv) exactly as EosSpec derives them (fluid.cpp:40-53)."""
    cpf, cvf = Fraction(*cp), Fraction(*cv)
    r = (cpf - cvf) / cvf
    g = cpf / cvf
    val = lambda f: float(f.numerator) / float(f.denominator)  # noqa: E731
    return val(r), val(g), val(cvf)


class Oracle:
    """The C restatement (fvb_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run make -C oracle")
        L = ctypes.CDLL(path)
        vp, u64, i32, dbl = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
        pp = ctypes.POINTER(ctypes.c_void_p)
        L.fvo_splitmix64_draw.restype = u64
        L.fvo_splitmix64_draw.argtypes = [u64, u64]
        L.fvo_uniform.restype = dbl
        L.fvo_uniform.argtypes = [u64, u64, dbl, dbl]
        for p in ("f64", "f32"):
            getattr(L, f"fvo_random_state_{p}").argtypes = [i32, u64, u64, u64, pp]
            getattr(L, f"fvo_make_vec_{p}").argtypes = [u64, u64, u64, dbl, dbl, vp]
            getattr(L, f"fvo_axpy_sin_{p}").argtypes = [u64, vp, vp]
            for fn in ("flux", "flux_prim", "cons2prim", "prim2cons"):
                getattr(L, f"fvo_{fn}_{p}").argtypes = [GasC, i32, u64, pp, pp]
            getattr(L, f"fvo_v_mag2_{p}").argtypes = [i32, u64, pp, vp]
            getattr(L, f"fvo_jacobian_{p}").argtypes = [GasC, i32, u64, pp, pp, vp]
        L.fvo_wave_speed_max_f64.restype = dbl
        L.fvo_wave_speed_max_f64.argtypes = [GasC, i32, u64, pp]
        L.fvo_wave_speed_max_f32.restype = ctypes.c_float
        L.fvo_wave_speed_max_f32.argtypes = [GasC, i32, u64, pp]
        L.fvo_wave_speed_f64.argtypes = [GasC, i32, u64, pp, vp]
        L.fvo_eos_p_f64.argtypes = [GasC, u64, vp, vp, vp]
        L.fvo_eos_T_f64.argtypes = [GasC, u64, vp, vp]
        L.fvo_eos_p_f32.argtypes = [GasC, u64, vp, vp, vp]
        L.fvo_eos_T_f32.argtypes = [GasC, u64, vp, vp]
        for yx in ("yd_xd", "yd_xs", "ys_xd", "ys_xs"):
            getattr(L, f"fvo_csr_matvec_acc_{yx}").argtypes = [u64, vp, vp, vp, vp, vp]
        self.L = L

    def csr_matvec_acc(self, rp, ci, v, x, y):
        """y += A x in y's precision, rows summed in stored order
        (block.cpp:345-356).  rp/ci uint64, v float64; returns the new y."""
        y = np.array(y, copy=True)
        yx = ("yd" if y.dtype == np.float64 else "ys") + "_" + \
             ("xd" if x.dtype == np.float64 else "xs")
        rp = np.ascontiguousarray(rp, np.uint64)
        ci = np.ascontiguousarray(ci, np.uint64)
        v = np.ascontiguousarray(v, np.float64)
        getattr(self.L, f"fvo_csr_matvec_acc_{yx}")(len(rp) - 1, rp.ctypes.data, ci.ctypes.data,
                                                     v.ctypes.data, x.ctypes.data, y.ctypes.data)
        return y

    @staticmethod
    def gas(cp=(7, 2), cv=(5, 2)) -> GasC:
        return GasC(*gas_constants(cp, cv))

    def draw(self, seed: int, k: int) -> int:
        return self.L.fvo_splitmix64_draw(seed, k)

    def random_state(self, dim, n, seed=0x5EED, first=0, prec="f64"):
        out = [np.empty(n, _DT[prec]) for _ in range(dim + 2)]
        getattr(self.L, f"fvo_random_state_{prec}")(dim, seed, first, n, _pp(out))
        return out

    def make_vec(self, seed, first, n, lo=0.25, hi=4.0, prec="f64"):
        out = np.empty(n, _DT[prec])
        getattr(self.L, f"fvo_make_vec_{prec}")(seed, first, n, lo, hi, out.ctypes.data)
        return out

    def axpy_sin(self, x, y):
        y = np.array(y, copy=True)
        getattr(self.L, f"fvo_axpy_sin_{_prec_of(x)}")(len(x), x.ctypes.data, y.ctypes.data)
        return y

    def _block(self, fn, dim, state, nout, gas):
        p = _prec_of(state[0])
        n = len(state[0])
        out = [np.empty(n, state[0].dtype) for _ in range(nout)]
        getattr(self.L, f"fvo_{fn}_{p}")(gas or self.gas(), dim, n, _pp(state), _pp(out))
        return out

    def flux(self, dim, state, gas=None):
        return self._block("flux", dim, state, (dim + 2) * dim, gas)

    def flux_prim(self, dim, prim, gas=None):
        return self._block("flux_prim", dim, prim, (dim + 2) * dim, gas)

    def cons2prim(self, dim, state, gas=None):
        return self._block("cons2prim", dim, state, dim + 2, gas)

    def prim2cons(self, dim, prim, gas=None):
        return self._block("prim2cons", dim, prim, dim + 1, gas)

    def v_mag2(self, dim, state):
        out = np.empty(len(state[0]), state[0].dtype)
        getattr(self.L, f"fvo_v_mag2_{_prec_of(state[0])}")(dim, len(out), _pp(state),
                                                            out.ctypes.data)
        return out

    def jacobian(self, dim, state, gas=None):
        p = _prec_of(state[0])
        n = len(state[0])
        w = dim + 2
        out = [np.empty(n, state[0].dtype) for _ in range(dim * w * w)]
        lam = np.zeros(1, state[0].dtype)
        getattr(self.L, f"fvo_jacobian_{p}")(gas or self.gas(), dim, n, _pp(state), _pp(out),
                                             lam.ctypes.data)
        return out, lam[0]

    def wave_speed_max(self, dim, state, gas=None):
        p = _prec_of(state[0])
        return getattr(self.L, f"fvo_wave_speed_max_{p}")(gas or self.gas(), dim, len(state[0]),
                                                          _pp(state))

    def wave_speed(self, dim, state, gas=None):
        out = np.empty(len(state[0]), np.float64)
        self.L.fvo_wave_speed_f64(gas or self.gas(), dim, len(out), _pp(state), out.ctypes.data)
        return out

    def eos(self, rho, e, gas=None):
        p = np.empty_like(rho)
        T = np.empty_like(rho)
        g = gas or self.gas()
        sfx = _prec_of(rho)
        getattr(self.L, f"fvo_eos_p_{sfx}")(g, len(rho), rho.ctypes.data, e.ctypes.data,
                                             p.ctypes.data)
        getattr(self.L, f"fvo_eos_T_{sfx}")(g, len(rho), e.ctypes.data, T.ctypes.data)
        return p, T


class Reference:
    """The unmodified reference, via ref_shim.cpp's C entry points."""

    def __init__(self, path: str = REF_SO):
        L = ctypes.CDLL(path)
        vp, u64, i32, dbl = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
        pp = ctypes.POINTER(ctypes.c_void_p)
        gas = ctypes.POINTER(ctypes.c_longlong)
        L.fvr_last_error.restype = ctypes.c_char_p
        L.fvr_hardware_threads.restype = ctypes.c_uint
        L.fvr_make_vec.argtypes = [u64, u64, u64, dbl, dbl, vp]
        L.fvr_random_state.argtypes = [i32, i32, u64, u64, pp]
        L.fvr_axpy_sin.argtypes = [i32, u64, vp, vp, i32]
        L.fvr_flux.argtypes = [gas, i32, i32, u64, pp, pp, i32]
        L.fvr_flux_prim.argtypes = [gas, i32, i32, u64, pp, pp, i32]
        L.fvr_cons2prim.argtypes = [gas, i32, i32, u64, pp, pp, i32]
        L.fvr_prim2cons.argtypes = [gas, i32, i32, u64, pp, pp, i32]
        L.fvr_v_mag2.argtypes = [i32, i32, u64, pp, vp, i32]
        L.fvr_eos.argtypes = [gas, i32, u64, vp, vp, vp, vp]
        L.fvr_jacobian.argtypes = [gas, i32, i32, u64, pp, pp, ctypes.POINTER(dbl), i32]
        L.fvr_wave_speed.argtypes = [gas, i32, i32, u64, pp, vp, ctypes.POINTER(dbl), i32]
        L.fvr_time_config.argtypes = [i32, i32, i32, u64, i32, i32, u64, ctypes.POINTER(dbl)]
        L.fvr_run_miniapp.argtypes = [i32, u64, i32, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]
        L.fvr_csr_matvec.argtypes = [i32, i32, i32, u64, u64, vp, vp, vp, vp, vp, vp]
        L.fvr_time_csr.argtypes = [u64, i32, ctypes.POINTER(dbl), ctypes.POINTER(u64)]
        self.L = L

    def csr_matvec(self, rp, ci, v, x, cols, y_prec="f64", m_prec="f64"):
        """y = A x through the reference's block_matvec / evaluate_block.
        Returns (y, the values as SparseMatrix stores them)."""
        rp = np.ascontiguousarray(rp, np.uint64)
        ci = np.ascontiguousarray(ci, np.uint64)
        v = np.ascontiguousarray(v, np.float64)
        rows = len(rp) - 1
        y = np.empty(rows, _DT[y_prec])
        stored = np.empty(len(v), np.float64)
        self._ok(self.L.fvr_csr_matvec(_PREC[y_prec], _PREC[_prec_of(x)], _PREC[m_prec], rows,
                                       cols, rp.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                       x.ctypes.data, y.ctypes.data, stored.ctypes.data))
        return y, stored

    def time_csr(self, n, reps):
        """Seconds per y = A x of the 7-point Laplacian on an n^3 grid
        (serial, as the reference's csr_matvec_acc is), and its nnz."""
        t = (ctypes.c_double * reps)()
        nnz = ctypes.c_uint64()
        self._ok(self.L.fvr_time_csr(n, reps, t, ctypes.byref(nnz)))
        return [x * 1e-9 for x in t], nnz.value

    def _ok(self, rc):
        if rc != 0:
            raise RuntimeError("reference: " + self.L.fvr_last_error().decode())

    @staticmethod
    def _gas(cp=(7, 2), cv=(5, 2)):
        return (ctypes.c_longlong * 4)(cp[0], cp[1], cv[0], cv[1])

    def hardware_threads(self) -> int:
        return int(self.L.fvr_hardware_threads())

    def make_vec(self, seed, first, n, lo=0.25, hi=4.0):
        out = np.empty(n, np.float64)
        self._ok(self.L.fvr_make_vec(seed, first, n, lo, hi, out.ctypes.data))
        return out

    def random_state(self, dim, n, seed=0x5EED, prec="f64"):
        out = [np.empty(n, _DT[prec]) for _ in range(dim + 2)]
        self._ok(self.L.fvr_random_state(dim, _PREC[prec], seed, n, _pp(out)))
        return out

    def axpy_sin(self, x, y, workers=0):
        y = np.array(y, copy=True)
        self._ok(self.L.fvr_axpy_sin(_PREC[_prec_of(x)], len(x), x.ctypes.data, y.ctypes.data,
                                     workers))
        return y

    def _block(self, fn, dim, state, nout, workers, cp, cv):
        n = len(state[0])
        out = [np.empty(n, state[0].dtype) for _ in range(nout)]
        self._ok(getattr(self.L, f"fvr_{fn}")(self._gas(cp, cv), dim, _PREC[_prec_of(state[0])],
                                              n, _pp(state), _pp(out), workers))
        return out

    def flux(self, dim, state, workers=0, cp=(7, 2), cv=(5, 2)):
        return self._block("flux", dim, state, (dim + 2) * dim, workers, cp, cv)

    def flux_prim(self, dim, prim, workers=0, cp=(7, 2), cv=(5, 2)):
        return self._block("flux_prim", dim, prim, (dim + 2) * dim, workers, cp, cv)

    def cons2prim(self, dim, state, workers=0, cp=(7, 2), cv=(5, 2)):
        return self._block("cons2prim", dim, state, dim + 2, workers, cp, cv)

    def prim2cons(self, dim, prim, workers=0, cp=(7, 2), cv=(5, 2)):
        return self._block("prim2cons", dim, prim, dim + 1, workers, cp, cv)

    def v_mag2(self, dim, state, workers=0):
        out = np.empty(len(state[0]), state[0].dtype)
        self._ok(self.L.fvr_v_mag2(dim, _PREC[_prec_of(state[0])], len(out), _pp(state),
                                   out.ctypes.data, workers))
        return out

    def eos(self, rho, e, cp=(7, 2), cv=(5, 2)):
        p = np.empty_like(rho)
        T = np.empty_like(rho)
        self._ok(self.L.fvr_eos(self._gas(cp, cv), _PREC[_prec_of(rho)], len(rho), rho.ctypes.data,
                                e.ctypes.data, p.ctypes.data, T.ctypes.data))
        return p, T

    def jacobian(self, dim, state, workers=0, cp=(7, 2), cv=(5, 2)):
        n = len(state[0])
        w = dim + 2
        out = [np.empty(n, state[0].dtype) for _ in range(dim * w * w)]
        lam = ctypes.c_double()
        self._ok(self.L.fvr_jacobian(self._gas(cp, cv), dim, _PREC[_prec_of(state[0])], n,
                                     _pp(state), _pp(out), ctypes.byref(lam), workers))
        return out, lam.value

    def wave_speed(self, dim, state, workers=0, cp=(7, 2), cv=(5, 2)):
        n = len(state[0])
        out = np.empty(n, state[0].dtype)
        lam = ctypes.c_double()
        self._ok(self.L.fvr_wave_speed(self._gas(cp, cv), dim, _PREC[_prec_of(state[0])], n,
                                       _pp(state), out.ctypes.data, ctypes.byref(lam), workers))
        return out, lam.value

    def time_config(self, which, dim, prec, n, workers, reps, seed=0x5EED):
        t = (ctypes.c_double * reps)()
        self._ok(self.L.fvr_time_config(which, dim, _PREC[prec], n, workers, reps, seed, t))
        return list(t)

    def run_miniapp(self, prec, n, workers):
        med, ratio = ctypes.c_double(), ctypes.c_double()
        self._ok(self.L.fvr_run_miniapp(_PREC[prec], n, workers, ctypes.byref(med),
                                        ctypes.byref(ratio)))
        return med.value, ratio.value


_oracle = None
_ref = None


def oracle() -> Oracle:
    global _oracle
    if _oracle is None:
        _oracle = Oracle()
    return _oracle


def reference():
    """The reference build, or None where it was not built."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = Reference()
    return _ref
