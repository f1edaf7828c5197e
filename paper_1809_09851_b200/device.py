"""Typed wrappers over the C ABI for torch CUDA tensors.

Planes are 1-D contiguous CUDA tensors (float32 or float64), one per field,
structure-of-arrays as in the reference (a conservative state is
``[rho, m_0..m_{d-1}, rhoE]``, proj/include/fusevec/fluid.hpp:81-88).  Every
call enqueues on the current torch stream (or ``stream=``) and returns
without synchronising.  Validation mirrors the reference's validate()
(proj/src/backend_eval.cpp:236-265): plane lengths must agree
(LengthMismatch) and precisions must be uniform (PrecisionError) before any
kernel is enqueued.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _native as N


@dataclass(frozen=True)
class Gas:
    """EosSpec(cp, cv) as rationals (proj/include/fusevec/fluid.hpp:27-45)."""

    cp_num: int = 7
    cp_den: int = 2
    cv_num: int = 5
    cv_den: int = 2

    @property
    def gamma_minus_one(self) -> float:
        # (R/cv).value() with R = cp - cv, both exact rationals (fluid.cpp:51-53)
        from fractions import Fraction
        cp, cv = Fraction(self.cp_num, self.cp_den), Fraction(self.cv_num, self.cv_den)
        r = (cp - cv) / cv
        return float(r.numerator) / float(r.denominator)

    @property
    def gamma(self) -> float:
        from fractions import Fraction
        g = Fraction(self.cp_num, self.cp_den) / Fraction(self.cv_num, self.cv_den)
        return float(g.numerator) / float(g.denominator)

    @property
    def cv(self) -> float:
        from fractions import Fraction
        c = Fraction(self.cv_num, self.cv_den)
        return float(c.numerator) / float(c.denominator)

    def struct(self) -> N.GasStruct:
        return N.GasStruct(self.gamma_minus_one, self.gamma, self.cv)


DEFAULT_GAS = Gas()

_PREC = {torch.float32: 0, torch.float64: 1}
_DTYPE = {0: torch.float32, 1: torch.float64}


def _gas_ptr(gas: Optional[Gas]):
    if gas is None:
        return None
    return ctypes.byref(gas.struct())


def _stream(stream, device=None) -> int:
    """The CUDA stream handle to enqueue on: `stream`, else the current torch
    stream of `device` (the planes' device), not of the current device."""
    if stream is None:
        return torch.cuda.current_stream(device).cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _scalar_out(t, prec: int, device, what: str) -> int:
    """Pointer of a caller-supplied lambda_max accumulator.  The kernel
    memsets and atomicMax-es one element of the state's precision there, so
    anything else (a CPU tensor, another GPU, a narrower dtype, no element)
    would be an out-of-bounds or foreign device write: refused up front."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise N.ArgumentError(N.FVB_EARG, f"{what}: must be a CUDA tensor")
    if t.device != torch.device(device):
        raise N.ArgumentError(N.FVB_EARG, f"{what}: on {t.device}, the state is on {device}")
    if t.dtype != _DTYPE[prec]:
        raise N.PrecisionError(N.FVB_EPREC, f"{what}: dtype {t.dtype}, the state is "
                                            f"{_DTYPE[prec]}")
    if t.numel() < 1:
        raise N.ArgumentError(N.FVB_EARG, f"{what}: needs one element")
    return t.data_ptr()


def _planes(planes: Sequence[torch.Tensor], what: str, n: Optional[int] = None,
            prec: Optional[int] = None, device=None):
    ptrs = []
    device = planes[0].device if device is None and len(planes) else device
    for t in planes:
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise N.ArgumentError(N.FVB_EARG, f"{what}: planes must be CUDA tensors")
        if t.device != device:
            raise N.ArgumentError(N.FVB_EARG, f"{what}: a plane on {t.device}, expected "
                                              f"{device}")
        if t.dim() != 1 or not t.is_contiguous():
            raise N.ArgumentError(N.FVB_EARG, f"{what}: planes must be contiguous 1-D")
        p = _PREC.get(t.dtype)
        if p is None:
            raise N.PrecisionError(N.FVB_EPREC, f"{what}: dtype {t.dtype} is not f32/f64")
        if prec is None:
            prec = p
        elif p != prec:
            raise N.PrecisionError(N.FVB_EPREC, f"{what}: mixed precisions")
        if n is None:
            n = t.numel()
        elif t.numel() != n:
            raise N.LengthMismatch(N.FVB_ELEN,
                                   f"{what}: plane length {t.numel()} does not match {n}")
        ptrs.append(t.data_ptr())
    return ptrs, n, prec


def _count(planes, count: int, what: str) -> None:
    """The C ABI reads exactly `count` plane pointers: a shorter list would
    hand it pointers from past the end of the array."""
    if len(planes) != count:
        raise N.ArgumentError(N.FVB_EARG, f"{what}: {count} planes expected, got {len(planes)}")


def _alloc(count: int, n: int, prec: int, device) -> list:
    return [torch.empty(n, dtype=_DTYPE[prec], device=device) for _ in range(count)]


def _state(state, dim):
    if len(state) != dim + 2:
        raise N.ArgumentError(N.FVB_EARG, f"a {dim}D state needs {dim + 2} planes, "
                                          f"got {len(state)}")
    return _planes(state, "state")


def flux(state: Sequence[torch.Tensor], dim: int, out=None, gas: Optional[Gas] = None,
         stream=None):
    """inviscid_flux of a conservative state: (d+2)*d planes, item r*d+c."""
    if out is not None:
        _count(out, (dim + 2) * dim, "flux out")
    ins, n, prec = _state(state, dim)
    if out is None:
        out = _alloc((dim + 2) * dim, n, prec, state[0].device)
    outs, _, _ = _planes(out, "flux out", n, prec, device=state[0].device)
    with torch.cuda.device(state[0].device):
        N.check(N.lib().fvb_flux(_gas_ptr(gas), dim, prec, n, N.ptr_array(ins), N.ptr_array(outs),
                                 _stream(stream, state[0].device)))
    return out


def flux_prim(prim, dim, out=None, gas=None, stream=None):
    """inviscid_flux of a primitive state [rho, v.., p] (fluid.cpp:290-298)."""
    if out is not None:
        _count(out, (dim + 2) * dim, "flux_prim out")
    ins, n, prec = _state(prim, dim)
    if out is None:
        out = _alloc((dim + 2) * dim, n, prec, prim[0].device)
    outs, _, _ = _planes(out, "flux_prim out", n, prec, device=prim[0].device)
    with torch.cuda.device(prim[0].device):
        N.check(N.lib().fvb_flux_prim(_gas_ptr(gas), dim, prec, n, N.ptr_array(ins),
                                      N.ptr_array(outs), _stream(stream, prim[0].device)))
    return out


def cons2prim(state, dim, out=None, gas=None, stream=None):
    """[v_0..v_{d-1}, p, c] of a conservative state."""
    if out is not None:
        _count(out, dim + 2, "cons2prim out")
    ins, n, prec = _state(state, dim)
    if out is None:
        out = _alloc(dim + 2, n, prec, state[0].device)
    outs, _, _ = _planes(out, "cons2prim out", n, prec, device=state[0].device)
    with torch.cuda.device(state[0].device):
        N.check(N.lib().fvb_cons2prim(_gas_ptr(gas), dim, prec, n, N.ptr_array(ins),
                                      N.ptr_array(outs), _stream(stream, state[0].device)))
    return out


def prim2cons(prim, dim, out=None, gas=None, stream=None):
    """[m_0..m_{d-1}, rhoE] of a primitive state [rho, v.., p]."""
    if out is not None:
        _count(out, dim + 1, "prim2cons out")
    ins, n, prec = _state(prim, dim)
    if out is None:
        out = _alloc(dim + 1, n, prec, prim[0].device)
    outs, _, _ = _planes(out, "prim2cons out", n, prec, device=prim[0].device)
    with torch.cuda.device(prim[0].device):
        N.check(N.lib().fvb_prim2cons(_gas_ptr(gas), dim, prec, n, N.ptr_array(ins),
                                      N.ptr_array(outs), _stream(stream, prim[0].device)))
    return out


def v_mag2(state, dim, out=None, stream=None):
    ins, n, prec = _state(state, dim)
    if out is None:
        out = _alloc(1, n, prec, state[0].device)[0]
    outs, _, _ = _planes([out], "v_mag2 out", n, prec, device=state[0].device)
    with torch.cuda.device(state[0].device):
        N.check(N.lib().fvb_v_mag2(dim, prec, n, N.ptr_array(ins), outs[0],
                                   _stream(stream, state[0].device)))
    return out


def eos(rho, e, p=None, T=None, gas=None, stream=None):
    """Ideal-gas closures: returns (p, T)."""
    ins, n, prec = _planes([rho, e], "eos")
    if p is None:
        p = _alloc(1, n, prec, rho.device)[0]
    if T is None:
        T = _alloc(1, n, prec, rho.device)[0]
    outs, _, _ = _planes([p, T], "eos out", n, prec, device=rho.device)
    with torch.cuda.device(rho.device):
        N.check(N.lib().fvb_eos(_gas_ptr(gas), prec, n, ins[0], ins[1], outs[0], outs[1],
                                _stream(stream, rho.device)))
    return p, T


def jacobian(state, dim, out=None, lambda_max=True, gas=None, stream=None):
    """Flux Jacobians [k][r][c] (d*(d+2)^2 planes) and, unless lambda_max is
    False, a 0-d device tensor holding the CFL max wave speed."""
    if out is not None:
        _count(out, dim * (dim + 2) ** 2, "jacobian out")
    ins, n, prec = _state(state, dim)
    w = dim + 2
    if out is None:
        out = _alloc(dim * w * w, n, prec, state[0].device)
    outs, _, _ = _planes(out, "jacobian out", n, prec, device=state[0].device)
    lam = None
    if lambda_max is True:
        lam = torch.empty((), dtype=_DTYPE[prec], device=state[0].device)
    elif lambda_max is not None and lambda_max is not False:
        lam = lambda_max
    lp = _scalar_out(lam, prec, state[0].device, "lambda_max") if lam is not None else None
    with torch.cuda.device(state[0].device):
        N.check(N.lib().fvb_jacobian(_gas_ptr(gas), dim, prec, n, N.ptr_array(ins),
                                     N.ptr_array(outs), lp, _stream(stream, state[0].device)))
    return out, lam


def wave_speed_max(state, dim, lam_out=None, lambda_max=None, gas=None, stream=None):
    """CFL reduction: returns (lambda per point or None, 0-d lambda_max)."""
    ins, n, prec = _state(state, dim)
    if lambda_max is None:
        lambda_max = torch.empty((), dtype=_DTYPE[prec], device=state[0].device)
    lp = None
    if lam_out is not None:
        lp = _planes([lam_out], "lambda out", n, prec, device=state[0].device)[0][0]
    with torch.cuda.device(state[0].device):
        N.check(N.lib().fvb_wave_speed_max(
            _gas_ptr(gas), dim, prec, n, N.ptr_array(ins), lp,
            _scalar_out(lambda_max, prec, state[0].device, "lambda_max"),
            _stream(stream, state[0].device)))
    return lam_out, lambda_max


def csr_matvec_acc(row_ptr, col_idx, values, x, y, stream=None):
    """y += A x for a CSR matrix (block.cpp:345-356): row_ptr (rows+1) int64
    and col_idx (nnz) int64 -- or int32, the narrow device layout
    (fvb_csr_matvec_acc_u32) -- CUDA tensors holding the unsigned indices,
    values float64 (already narrowed to the matrix precision); x and y
    f32/f64 planes.  Each row is summed in stored order in y's precision."""
    if not row_ptr.is_cuda or row_ptr.dtype != torch.int64 or row_ptr.dim() != 1:
        raise N.ArgumentError(N.FVB_EARG, "row_ptr must be a 1-D int64 CUDA tensor")
    if not col_idx.is_cuda or col_idx.dtype not in (torch.int64, torch.int32) or col_idx.dim() != 1:
        raise N.ArgumentError(N.FVB_EARG, "col_idx must be a 1-D int64 or int32 CUDA tensor")
    if not values.is_cuda or values.dtype != torch.float64 or values.numel() != col_idx.numel():
        raise N.ArgumentError(N.FVB_EARG, "values must be float64 with one entry per index")
    (xp,), cols, px = _planes([x], "x")
    (yp,), rows, py = _planes([y], "y", device=x.device)
    if row_ptr.numel() != rows + 1:
        raise N.LengthMismatch(N.FVB_ELEN, f"row_ptr has {row_ptr.numel()} entries for "
                                           f"{rows} rows")
    if any(t.device != y.device for t in (row_ptr, col_idx, values)):
        raise N.ArgumentError(N.FVB_EARG, "CSR arrays must be on the planes' device")
    fn = N.lib().fvb_csr_matvec_acc_u32 if col_idx.dtype == torch.int32 else \
        N.lib().fvb_csr_matvec_acc
    with torch.cuda.device(y.device):
        N.check(fn(py, px, rows, col_idx.numel(), row_ptr.data_ptr(), col_idx.data_ptr(),
                   values.data_ptr(), xp, yp, _stream(stream, y.device)))
    return y


def axpy_sin(x, y, stream=None):
    """y <- 0.5*sin(x+y) in place."""
    ptrs, n, prec = _planes([x, y], "axpy_sin")
    with torch.cuda.device(y.device):
        N.check(N.lib().fvb_axpy_sin(prec, n, ptrs[0], ptrs[1], _stream(stream, y.device)))
    return y


def synth_state(dim, n, prec=1, seed=0x5EED, first=0, out=None, device="cuda", stream=None):
    """random_state of acceptance.cpp:214-230 for global points [first, first+n)."""
    if out is None:
        out = _alloc(dim + 2, n, prec, device)
    _count(out, dim + 2, "synth out")
    # the generator writes planes of `prec`: their dtype and length must match
    outs, _, _ = _planes(out, "synth out", n, prec) if n else ([0] * (dim + 2), 0, prec)
    with torch.cuda.device(out[0].device if n else device):
        N.check(N.lib().fvb_synth_state(dim, prec, seed, first, n, N.ptr_array(outs),
                                        _stream(stream, out[0].device if n else device)))
    return out


def synth_uniform(n, prec=1, seed=1, first=0, lo=0.25, hi=4.0, out=None, device="cuda",
                  stream=None):
    """make_vec of oracle.hpp:118-123: uniform(lo, hi) of draws [first, first+n)."""
    if out is None:
        out = _alloc(1, n, prec, device)[0]
    ptr = _planes([out], "synth_uniform out", n, prec)[0][0] if n else None
    with torch.cuda.device(out.device):
        N.check(N.lib().fvb_synth_uniform(prec, seed, first, n, lo, hi, ptr,
                                          _stream(stream, out.device)))
    return out


def patterns():
    """[(name, pattern key)] of every registered fused kernel."""
    L = N.lib()
    out = []
    for i in range(L.fvb_pattern_count()):
        name = ctypes.c_char_p()
        text = L.fvb_pattern(i, ctypes.byref(name))
        out.append((name.value.decode(), text.decode()))
    return out


def lookup(key: str) -> N.KernelStruct:
    """fvb_lookup: the fused kernel for a structural key (raises
    UnsupportedExpression when none exists)."""
    k = N.KernelStruct()
    N.check(N.lib().fvb_lookup(key.encode(), ctypes.byref(k)))
    return k


def emit_source(key: str) -> str:
    """The CUDA source the general lowering compiles for a structural key."""
    n = ctypes.c_size_t()
    N.check(N.lib().fvb_emit_source(key.encode(), None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    N.check(N.lib().fvb_emit_source(key.encode(), buf, n.value + 1, ctypes.byref(n)))
    return buf.value.decode()


def nvrtc_compile(key: str) -> int:
    """Compile a key's lowered kernel with NVRTC (no GPU needed); cubin bytes."""
    n = ctypes.c_size_t()
    N.check(N.lib().fvb_nvrtc_compile(key.encode(), ctypes.byref(n)))
    return n.value


class HostContext:
    """fvb_ctx: the host-buffer (end-to-end) path over pinned/pageable memory."""

    def __init__(self, device: int = 0, chunk_points: int = 0):
        self._h = ctypes.c_void_p()
        N.check(N.lib().fvb_ctx_create(device, chunk_points, ctypes.byref(self._h)))

    def close(self):
        if self._h:
            N.lib().fvb_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _host(planes, what, n=None, prec=None):
        ptrs = []
        for t in planes:
            if t.is_cuda or t.dim() != 1 or not t.is_contiguous():
                raise N.ArgumentError(N.FVB_EARG, f"{what}: host planes must be CPU 1-D")
            p = _PREC[t.dtype]
            prec = p if prec is None else prec
            if p != prec:
                raise N.PrecisionError(N.FVB_EPREC, f"{what}: mixed precisions")
            n = t.numel() if n is None else n
            if t.numel() != n:
                raise N.LengthMismatch(N.FVB_ELEN, f"{what}: ragged planes")
            ptrs.append(t.data_ptr())
        return ptrs, n, prec

    def flux(self, state, dim, out, gas=None):
        _count(state, dim + 2, "state")
        _count(out, (dim + 2) * dim, "flux out")
        ins, n, prec = self._host(state, "state")
        outs, _, _ = self._host(out, "out", n, prec)
        N.check(N.lib().fvb_flux_host(self._h, _gas_ptr(gas), dim, prec, n, N.ptr_array(ins),
                                      N.ptr_array(outs)))
        return out

    def launch(self, kernel, planes, n, reduce=False, after=None):
        """fvb_launch_host: run a structural-key kernel (lookup()) over
        `planes` -- its argument block, outputs then leaves in slot order.
        Each plane is a 1-D tensor (CPU: pinned or pageable; CUDA: used in
        place) or None for a NULL output slot.  Returns lambda_max when
        `reduce` (the kernel's CFL reduction)."""
        count = kernel.n_outputs + kernel.n_inputs
        if len(planes) != count:
            raise N.ArgumentError(N.FVB_EARG, f"kernel takes {count} planes, got {len(planes)}")
        ptrs, prec, dev = [], [], []
        for t in planes:
            if t is None:
                ptrs.append(0)
                prec.append(1)
                dev.append(0)
                continue
            if t.dim() != 1 or not t.is_contiguous() or t.numel() != n:
                raise N.ArgumentError(N.FVB_EARG, "planes must be contiguous 1-D of length n")
            ptrs.append(t.data_ptr())
            prec.append(_PREC[t.dtype])
            dev.append(1 if t.is_cuda else 0)
        lam = ctypes.c_double()
        N.check(N.lib().fvb_launch_host(
            self._h, ctypes.byref(kernel), n, N.ptr_array(ptrs), (ctypes.c_uint8 * count)(*prec),
            (ctypes.c_uint8 * count)(*dev), ctypes.byref(lam) if reduce else None,
            _stream(after) if after is not None else None))
        return lam.value if reduce else None

    def jacobian(self, state, dim, out, gas=None):
        _count(state, dim + 2, "state")
        _count(out, dim * (dim + 2) ** 2, "jacobian out")
        ins, n, prec = self._host(state, "state")
        outs, _, _ = self._host(out, "out", n, prec)
        lam = ctypes.c_double()
        N.check(N.lib().fvb_jacobian_host(self._h, _gas_ptr(gas), dim, prec, n,
                                          N.ptr_array(ins), N.ptr_array(outs),
                                          ctypes.byref(lam)))
        return out, lam.value
