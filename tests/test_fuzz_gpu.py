"""Randomised parity sweep over the C ABI: a few hundred seeded cases of
random block, dimension, precision, gas, length (around every launch-shape
threshold: the scalar head/tail, the 64-thread small-range shape, the
one-shot tile grid) and per-plane element offsets (mixed 32-byte residues),
each bitwise against the oracle.  Seeded, so a failure reproduces."""

import numpy as np
import pytest
import torch

import paper_1809_09851_b200 as fvb

pytestmark = pytest.mark.gpu

DT = {"f64": torch.float64, "f32": torch.float32}
GASES = [((7, 2), (5, 2)), ((5, 2), (3, 2)), ((13, 3), (11, 5))]
# the small-range threshold is SMs * 256 * (32 B / element size)
SIZES = [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 63, 64, 65, 255, 256, 257, 1023, 1024, 1025,
         4095, 4097, 37_887, 37_889, 75_775, 75_777, 151_551, 151_553, 303_103, 303_105,
         600_001]


def planes_at(arrs, offsets, dev):
    out = []
    for a, off in zip(arrs, offsets):
        buf = torch.empty(len(a) + 8, dtype=torch.from_numpy(a[:0]).dtype, device=dev)
        v = buf[off:off + len(a)]
        v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        out.append(v)
    return out


def empties(count, n, dt, offsets, dev):
    return [torch.empty(n + 8, dtype=dt, device=dev)[o:o + n] for o in offsets[:count]]


def same(ts, want):
    torch.cuda.synchronize()
    return all(t.cpu().numpy().tobytes() == np.asarray(w).tobytes() for t, w in zip(ts, want))


@pytest.mark.parametrize("chunk", range(6))
def test_random_cases_bitwise(cuda, orc, chunk):
    rng = np.random.default_rng(1000 + chunk)
    for case in range(50):
        block = rng.choice(["flux", "flux_prim", "cons2prim", "prim2cons", "v_mag2", "jacobian",
                            "wave_speed"])
        dim = int(rng.integers(1, 4))
        prec = "f64" if rng.random() < 0.5 else "f32"
        n = int(rng.choice(SIZES))
        cp, cv = GASES[int(rng.integers(0, len(GASES)))]
        gas, og = fvb.Gas(cp[0], cp[1], cv[0], cv[1]), orc.gas(cp=cp, cv=cv)
        offsets = [int(x) for x in rng.integers(0, 8, 100)]
        if rng.random() < 0.5:  # all planes on one residue: the vector path
            offsets = [offsets[0]] * 100
        s_np = orc.random_state(dim, n, seed=int(rng.integers(1, 1 << 30)), prec=prec)
        s = planes_at(s_np, offsets, cuda)
        outs_at = offsets[dim + 2:]
        what = (block, dim, prec, n, cp, cv, offsets[:4])
        w = dim + 2
        if block == "flux":
            out = empties(w * dim, n, DT[prec], outs_at, cuda)
            fvb.flux(s, dim, out=out, gas=gas)
            assert same(out, orc.flux(dim, s_np, gas=og)), what
        elif block == "flux_prim":
            out = empties(w * dim, n, DT[prec], outs_at, cuda)
            fvb.flux_prim(s, dim, out=out, gas=gas)
            assert same(out, orc.flux_prim(dim, s_np, gas=og)), what
        elif block == "cons2prim":
            out = empties(w, n, DT[prec], outs_at, cuda)
            fvb.cons2prim(s, dim, out=out, gas=gas)
            assert same(out, orc.cons2prim(dim, s_np, gas=og)), what
        elif block == "prim2cons":
            out = empties(dim + 1, n, DT[prec], outs_at, cuda)
            fvb.prim2cons(s, dim, out=out, gas=gas)
            assert same(out, orc.prim2cons(dim, s_np, gas=og)), what
        elif block == "v_mag2":
            out = empties(1, n, DT[prec], outs_at, cuda)
            fvb.v_mag2(s, dim, out=out[0])
            assert same(out, [orc.v_mag2(dim, s_np)]), what
        elif block == "jacobian":
            out = empties(dim * w * w, n, DT[prec], (outs_at * 4)[:dim * w * w], cuda)
            _, lam = fvb.jacobian(s, dim, out=out, gas=gas)
            j_np, lam_np = orc.jacobian(dim, s_np, gas=og)
            assert same(out, j_np), what
            assert lam.item() == float(lam_np), what
        else:
            lam_pts = empties(1, n, DT[prec], outs_at, cuda)[0]
            _, lam = fvb.wave_speed_max(s, dim, lam_out=lam_pts, gas=gas)
            _, lam_np = orc.jacobian(dim, s_np, gas=og)
            torch.cuda.synchronize()
            assert lam.item() == float(lam_np) == lam_pts.max().item(), what


@pytest.mark.parametrize("chunk", range(2))
def test_random_host_buffer_cases_bitwise(cuda, orc, chunk):
    # The host-buffer (end-to-end) path: random dimension, precision, gas,
    # length, staging chunk (so chunks end anywhere: ragged last chunks,
    # one-chunk ranges), pinned or pageable planes; the flux's host-side
    # row-0 copies and the Jacobian's host-side constant fills included.
    # Outputs start as NaN so a skipped host-side write shows.
    rng = np.random.default_rng(2000 + chunk)
    for case in range(20):
        block = rng.choice(["flux", "jacobian"])
        dim = int(rng.integers(1, 4))
        prec = "f64" if rng.random() < 0.5 else "f32"
        n = int(rng.choice([1, 7, 255, 257, 4097, 75_777, 300_001]))
        cp, cv = GASES[int(rng.integers(0, len(GASES)))]
        gas, og = fvb.Gas(cp[0], cp[1], cv[0], cv[1]), orc.gas(cp=cp, cv=cv)
        pinned = bool(rng.random() < 0.5)
        ctx = fvb.HostContext(0, chunk_points=int(rng.choice([256, 1024, 65_536, 0])))
        s_np = orc.random_state(dim, n, seed=int(rng.integers(1, 1 << 30)), prec=prec)
        hs = [torch.from_numpy(a) for a in s_np]
        count = (dim + 2) * dim if block == "flux" else dim * (dim + 2) ** 2
        outs = [torch.full((n,), float("nan"), dtype=DT[prec]) for _ in range(count)]
        if pinned:
            hs = [t.pin_memory() for t in hs]
            outs = [t.pin_memory() for t in outs]
        what = (block, dim, prec, n, cp, cv, pinned)
        if block == "flux":
            ctx.flux(hs, dim, outs, gas=gas)
            want = orc.flux(dim, s_np, gas=og)
        else:
            _, lam = ctx.jacobian(hs, dim, outs, gas=gas)
            want, lam_w = orc.jacobian(dim, s_np, gas=og)
            assert lam == lam_w, what
        assert all(o.numpy().tobytes() == np.asarray(w).tobytes() for o, w in zip(outs, want)), what
        ctx.close()
