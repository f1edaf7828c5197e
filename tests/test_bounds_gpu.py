"""Bounds: every device entry point at small, ragged, offset sizes with
guard bands around every plane.

compute-sanitizer is not available on the GPU pool, so out-of-range stores
are caught directly: each plane lives inside its own allocation between two
guard bands (longer than one 32-byte access) filled with a sentinel bit
pattern, and after every call the bands must be untouched and the input
planes unchanged.  Sizes cover the scalar head, the vector body and the
scalar tail; element offsets cover unaligned planes and mixed residues.
Results are compared with the oracle as well.
"""

import ctypes
import re
import struct

import numpy as np
import pytest
import torch

import paper_1809_09851_b200 as fvb
from paper_1809_09851_b200 import _native as N

pytestmark = pytest.mark.gpu

DT = {0: torch.float32, 1: torch.float64}
IT = {0: torch.int32, 1: torch.int64}
SENT = {0: 0x7FA5A5A5, 1: 0x7FF5A5A5A5A5A5A5}  # signalling-NaN sentinels
GUARD = 80  # elements per band: > one 256-bit access in either precision


class Arena:
    """Planes with guard bands; check() verifies every band and input."""

    def __init__(self, dev):
        self.dev = dev
        self.bufs = []    # (buffer, lo, hi, prec)
        self.inputs = []  # (plane, saved copy)

    def plane(self, n, prec, off=0):
        buf = torch.empty(2 * GUARD + off + n, dtype=DT[prec], device=self.dev)
        buf.view(IT[prec]).fill_(SENT[prec])
        lo = GUARD + off
        self.bufs.append((buf, lo, lo + n, prec))
        return buf[lo:lo + n]

    def planes(self, count, n, prec, off=0):
        return [self.plane(n, prec, off) for _ in range(count)]

    def inputs_from(self, arrs, off=0):
        out = []
        for a in arrs:
            prec = 1 if a.dtype == np.float64 else 0
            t = self.plane(len(a), prec, off)
            t.copy_(torch.from_numpy(np.ascontiguousarray(a)))
            out.append(t)
            self.inputs.append((t, t.clone()))
        return out

    def check(self, what):
        torch.cuda.synchronize()
        for buf, lo, hi, prec in self.bufs:
            bits = buf.view(IT[prec])
            assert bool((bits[:lo] == SENT[prec]).all()), f"{what}: store before a plane"
            assert bool((bits[hi:] == SENT[prec]).all()), f"{what}: store past a plane"
        for t, saved in self.inputs:
            assert torch.equal(t.view(IT[1 if t.dtype == torch.float64 else 0]),
                               saved.view(IT[1 if t.dtype == torch.float64 else 0])), \
                f"{what}: an input plane changed"


def bits_equal(ts, want):
    torch.cuda.synchronize()
    return all(t.cpu().numpy().tobytes() == np.asarray(w).tobytes() for t, w in zip(ts, want))


def hexbits(v):
    return "%016x" % struct.unpack("<Q", struct.pack("<d", v))[0]


@pytest.mark.parametrize("prec,p", [(1, "f64"), (0, "f32")])
@pytest.mark.parametrize("n", [1, 7, 33, 4099])
@pytest.mark.parametrize("off", [0, 1, 3])
def test_fluid_entry_points_stay_in_bounds(cuda, orc, prec, p, n, off):
    for dim in (1, 2, 3):
        A = Arena(cuda)
        s_np = orc.random_state(dim, n, seed=n + off, prec=p)
        s = A.inputs_from(s_np, off)
        w = dim + 2
        out = A.planes(w * dim, n, prec, off)
        fvb.flux(s, dim, out=out)
        assert bits_equal(out, orc.flux(dim, s_np))
        fvb.flux_prim(s, dim, out=A.planes(w * dim, n, prec, off))
        out = A.planes(w, n, prec, off)
        fvb.cons2prim(s, dim, out=out)
        assert bits_equal(out, orc.cons2prim(dim, s_np))
        fvb.prim2cons(s, dim, out=A.planes(dim + 1, n, prec, off))
        fvb.v_mag2(s, dim, out=A.plane(n, prec, off))
        out = A.planes(dim * w * w, n, prec, off)
        _, lam = fvb.jacobian(s, dim, out=out)
        jw, lw = orc.jacobian(dim, s_np)
        assert bits_equal(out, jw) and lam.item() == lw
        _, lam2 = fvb.wave_speed_max(s, dim, lam_out=A.plane(n, prec, off))
        _, lam3 = fvb.wave_speed_max(s, dim)
        assert lam2.item() == lam3.item() == lw
        A.check(f"fluid d={dim}")
    A = Arena(cuda)
    rho, e = A.inputs_from([orc.make_vec(1, 0, n, prec=p), orc.make_vec(2, 0, n, prec=p)], off)
    fvb.eos(rho, e, p=A.plane(n, prec, off), T=A.plane(n, prec, off))
    x = A.inputs_from([orc.make_vec(1, 0, n, prec=p)], off)[0]
    y = A.plane(n, prec, off)
    y.copy_(torch.from_numpy(orc.make_vec(1, n, n, prec=p)))
    fvb.axpy_sin(x, y)
    fvb.synth_state(3, n, prec=prec, first=off, out=A.planes(5, n, prec, off))
    fvb.synth_uniform(n, prec=prec, out=A.plane(n, prec, off))
    A.check("eos/axpy/synth")


def test_structural_key_kernels_stay_in_bounds(cuda, orc):
    A = Arena(cuda)
    n = 4099
    s_np = orc.random_state(3, n, seed=3)
    s = A.inputs_from(s_np, 1)
    vals = {"half": 0.5, "gm1": 0.4, "gamma": 1.4, "zero": 0.0, "one": 1.0, "cv": 2.5}
    stream = torch.cuda.current_stream().cuda_stream
    for name in ("flux3_f64", "jacobian3_f64"):
        pat = dict(fvb.patterns())[name]
        k = fvb.lookup(re.sub(r"Cd#(\w+);", lambda m: "Cd" + hexbits(vals[m.group(1)]) + ";",
                              pat))
        slots = [None] * k.n_inputs
        for ci in range(k.n_inputs):
            slots[k.in_slot[ci]] = s[ci]
        outs = A.planes(k.n_outputs, n, 1)
        args = N.ptr_array([t.data_ptr() for t in outs + slots])
        for b, e in ((0, 1000), (1000, n)):  # split ranges, as JitKernel::Fn
            N.check(k.fn(ctypes.byref(k), b, e, args, stream))
    # lowered kernels, vector body (offset 0) and element path (offset 1);
    # argument precisions are outputs, then leaf slots
    for key, precs in (("dB4d(U11d(Ld0;),B7d(Ld1;,U20d(Ld0;)))", (1, 1, 1)),
                       ("G1x2:sU8s(Ls0;)|dU10d(B3d(Ld1;,Cd" + hexbits(3.0) + ";))",
                        (0, 1, 0, 1))):
        k = fvb.lookup(key)
        assert k.n_outputs + k.n_inputs == len(precs)
        for off in (0, 1):
            a = [A.plane(n, q, off) for q in precs]
            for t in a:
                t.uniform_(0.5, 2.0)
            args = N.ptr_array([t.data_ptr() for t in a])
            N.check(k.fn(ctypes.byref(k), 0, n, args, stream))
    A.check("structural-key kernels")


@pytest.mark.parametrize("idx", ["u64", "u32"])
@pytest.mark.parametrize("mode", ["row", "warp"])
def test_csr_matvec_stays_in_bounds(cuda, mode, idx, monkeypatch):
    monkeypatch.setenv("FVB_CSR_MODE", mode)
    A = Arena(cuda)
    rows, cols = 257, 301
    rng = np.random.default_rng(0)
    rp = np.zeros(rows + 1, np.uint64)
    ci, vv = [], []
    for r in range(rows):
        c = np.sort(rng.choice(cols, rng.integers(0, 6), replace=False))
        ci += list(c)
        vv += list(rng.uniform(-1, 1, len(c)))
        rp[r + 1] = len(ci)
    drp = torch.from_numpy(rp.view(np.int64)).to(cuda)
    # values and indices in guarded planes too, one element off a 16-byte
    # boundary, checked unchanged after
    dv = A.inputs_from([np.array(vv)], 1)[0]
    if idx == "u64":
        dci = A.plane(len(ci), 1, 3)
        dci.view(torch.int64).copy_(torch.from_numpy(np.array(ci, np.uint64).view(np.int64)))
    else:  # 32-bit indices, 4 bytes off a 16-byte boundary
        dci = A.plane(len(ci), 0, 1)
        dci.view(torch.int32).copy_(torch.from_numpy(np.array(ci, np.int32)))
    A.inputs.append((dci, dci.clone()))
    fn = N.lib().fvb_csr_matvec_acc if idx == "u64" else N.lib().fvb_csr_matvec_acc_u32
    xh = rng.uniform(-1, 1, cols)
    x = A.inputs_from([xh], 1)[0]
    y = A.plane(rows, 1, 3)
    y.zero_()
    N.check(fn(1, 1, rows, len(ci), drp.data_ptr(), dci.data_ptr(), dv.data_ptr(), x.data_ptr(),
               y.data_ptr(), torch.cuda.current_stream().cuda_stream))
    # csr_matvec_acc_t (proj/src/block.cpp:345-356): acc in stored order, y += acc
    want = np.zeros(rows)
    for r in range(rows):
        acc = np.float64(0.0)
        for k in range(int(rp[r]), int(rp[r + 1])):
            acc = acc + np.float64(vv[k]) * np.float64(xh[ci[k]])
        want[r] = want[r] + acc
    A.check("csr")
    assert y.cpu().numpy().tobytes() == want.tobytes()


def test_host_pipeline_multi_chunk(cuda, orc):
    # several chunks per slot: the staging offsets of every chunk
    ctx = fvb.HostContext(0, chunk_points=1024)
    for dim in (1, 3):
        s_np = orc.random_state(dim, 5001, seed=9)
        hin = [torch.from_numpy(a) for a in s_np]
        hout = [torch.empty(5001, dtype=torch.float64) for _ in range((dim + 2) * dim)]
        ctx.flux(hin, dim, hout)
        assert all(h.numpy().tobytes() == w.tobytes() for h, w in zip(hout, orc.flux(dim, s_np)))
        jout = [torch.empty(5001, dtype=torch.float64) for _ in range(dim * (dim + 2) ** 2)]
        _, lam = ctx.jacobian(hin, dim, jout)
        jw, lw = orc.jacobian(dim, s_np)
        assert lam == lw
        assert all(h.numpy().tobytes() == w.tobytes() for h, w in zip(jout, jw))
    ctx.close()
