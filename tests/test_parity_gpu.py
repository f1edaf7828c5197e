"""Device parity: every kernel of libfvb.so against the CPU oracle (which
tests/test_oracle.py pins to the reference bit for bit).

Bars (BASELINE.json north_star): bitwise for +,-,*,/,sqrt (the whole fluid
path: flux, cons->prim, EOS, Jacobians, wave speed) and for the synthetic
generators; the CFL maximum exactly; sin within 4 ulp (f64) / rel 1e-6
(f32).  Runs only on a B200 (`-m gpu`), through the C ABI.
"""

import ctypes
import os

import numpy as np
import pytest
import torch

import paper_1809_09851_b200 as fvb
from paper_1809_09851_b200 import _native as N

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
DT = {"f64": torch.float64, "f32": torch.float32}
NP = {"f64": np.float64, "f32": np.float32}
PREC = {"f32": 0, "f64": 1}
SIZES = [0, 1, 2, 3, 5, 7, 8, 31, 1023, 1025, 4099, 65537]


def to_dev(arrs, dev):
    return [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in arrs]


def to_host(ts):
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in ts]


def same_bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


def all_same(xs, ys):
    return len(xs) == len(ys) and all(same_bits(x, y) for x, y in zip(xs, ys))


def ulp_diff(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    ia = a.view(np.int64)
    ib = b.view(np.int64)
    ia = np.where(ia < 0, np.int64(-0x8000000000000000) - ia, ia)
    ib = np.where(ib < 0, np.int64(-0x8000000000000000) - ib, ib)
    return np.abs(ia - ib)


# ---- synthetic inputs ---------------------------------------------------------


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_synth_state_bitwise(cuda, orc, prec, dim):
    for n, first in [(1, 0), (1000, 0), (4099, 123456789)]:
        dev = fvb.synth_state(dim, n, prec=PREC[prec], seed=0x5EED, first=first)
        want = orc.random_state(dim, n, seed=0x5EED, first=first, prec=prec)
        assert all_same(to_host(dev), want)


def test_synth_outputs_are_validated(cuda):
    # the generators write planes of `prec`: an f32 plane (half the bytes)
    # or a short plane under prec=1 would be an out-of-bounds device write
    with pytest.raises(fvb.PrecisionError):
        fvb.synth_state(3, 100, prec=1, out=[torch.empty(100, dtype=torch.float32, device=cuda)
                                             for _ in range(5)])
    with pytest.raises(fvb.LengthMismatch):
        fvb.synth_state(3, 100, prec=1, out=[torch.empty(99, dtype=torch.float64, device=cuda)
                                             for _ in range(5)])
    with pytest.raises(fvb.PrecisionError):
        fvb.synth_uniform(100, prec=1, out=torch.empty(100, dtype=torch.float32, device=cuda))
    with pytest.raises(fvb.LengthMismatch):
        fvb.synth_uniform(100, prec=0, out=torch.empty(50, dtype=torch.float32, device=cuda))


def test_misaligned_device_planes_refused_before_launch(cuda, orc):
    # a misaligned plane would be a sticky device fault (the context dies):
    # the generators and the CSR accumulation refuse it with FVB_EALIGN, and
    # the device keeps working afterwards
    raw = torch.empty(8 * 1000 + 8, dtype=torch.uint8, device=cuda)
    odd = raw.data_ptr() + 4
    planes = [torch.empty(1000, dtype=torch.float64, device=cuda) for _ in range(5)]
    ptrs = [t.data_ptr() for t in planes]
    ptrs[2] = odd
    assert N.lib().fvb_synth_state(3, 1, 5, 0, 1000, N.ptr_array(ptrs), None) == N.FVB_EALIGN
    assert N.lib().fvb_synth_uniform(1, 5, 0, 1000, 0.0, 1.0, odd, None) == N.FVB_EALIGN
    rp, ci, v = stencil7(5)
    drp, dci, dv = _csr_to_dev(rp, ci, v, cuda)
    x = torch.zeros(len(rp) - 1, dtype=torch.float64, device=cuda)
    st = N.lib().fvb_csr_matvec_acc(1, 1, len(rp) - 1, len(ci), drp.data_ptr(), dci.data_ptr(),
                                    dv.data_ptr(), x.data_ptr(), odd, None)
    assert st == N.FVB_EALIGN
    torch.cuda.synchronize()
    s = fvb.synth_state(3, 1000)
    assert all_same(to_host(s), orc.random_state(3, 1000, seed=0x5EED))


def test_synth_uniform_bitwise(cuda, orc):
    for prec in ("f64", "f32"):
        d = fvb.synth_uniform(3000, prec=PREC[prec], seed=1, first=3000)
        assert same_bits(to_host([d])[0], orc.make_vec(1, 3000, 3000, prec=prec))


# ---- fluid blocks, bitwise ----------------------------------------------------------


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_fluid_blocks_bitwise(cuda, orc, prec, dim):
    for n in SIZES:
        s_np = orc.random_state(dim, n, seed=0xF1 + n, prec=prec)
        s = to_dev(s_np, cuda)
        assert all_same(to_host(fvb.flux(s, dim)), orc.flux(dim, s_np)), ("flux", n)
        c = to_host(fvb.cons2prim(s, dim))
        assert all_same(c, orc.cons2prim(dim, s_np)), ("cons2prim", n)
        prim_np = [s_np[0]] + c[:dim] + [c[dim]]
        assert all_same(to_host(fvb.prim2cons(to_dev(prim_np, cuda), dim)),
                        orc.prim2cons(dim, prim_np)), ("prim2cons", n)
        assert all_same(to_host(fvb.flux_prim(to_dev(prim_np, cuda), dim)),
                        orc.flux_prim(dim, prim_np)), ("flux_prim", n)
        assert same_bits(to_host([fvb.v_mag2(s, dim)])[0], orc.v_mag2(dim, s_np))
        j, lam = fvb.jacobian(s, dim)
        j_np, lam_np = orc.jacobian(dim, s_np)
        assert all_same(to_host(j), j_np), ("jacobian", n)
        assert same_bits(lam.cpu().numpy(), np.asarray(lam_np)), ("lambda", n)
        _, lam2 = fvb.wave_speed_max(s, dim)
        assert same_bits(lam2.cpu().numpy(), np.asarray(lam_np))


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_golden_fixtures(cuda, prec, dim):
    z = np.load(os.path.join(GOLDEN, f"fluid_{prec}_d{dim}.npz"))
    s = to_dev(list(z["state"]), cuda)
    assert same_bits(np.stack(to_host(fvb.flux(s, dim))), z["flux"])
    assert same_bits(np.stack(to_host(fvb.cons2prim(s, dim))), z["cons2prim"])
    assert same_bits(np.stack(to_host(fvb.prim2cons(to_dev(list(z["prim"]), cuda), dim))),
                     z["prim2cons"])
    assert same_bits(to_host([fvb.v_mag2(s, dim)])[0], z["v_mag2"])
    j, lam = fvb.jacobian(s, dim)
    assert same_bits(np.stack(to_host(j)), z["jacobian"])
    assert float(lam.item()) == float(z["lambda_max"])
    lam_pts = torch.empty_like(s[0])
    fvb.wave_speed_max(s, dim, lam_out=lam_pts)
    assert same_bits(to_host([lam_pts])[0], z["wave_speed"])


def test_golden_eos_and_monatomic(cuda):
    z = np.load(os.path.join(GOLDEN, "eos.npz"))
    p, T = fvb.eos(*to_dev([z["rho"], z["e"]], cuda))
    assert same_bits(p.cpu().numpy(), z["p"]) and same_bits(T.cpu().numpy(), z["T"])
    mono = fvb.Gas(5, 2, 3, 2)
    p, T = fvb.eos(*to_dev([z["rho"], z["e"]], cuda), gas=mono)
    assert same_bits(p.cpu().numpy(), z["p_mono"]) and same_bits(T.cpu().numpy(), z["T_mono"])
    c = fvb.cons2prim(to_dev(list(z["mono_state"]), cuda), 1, gas=mono)
    assert same_bits(np.stack(to_host(c)), z["mono_cons2prim"])
    assert c[1].item() == 2.0  # test_fluid.cpp:347-353


def test_gas_variant_bitwise(cuda, orc):
    g = fvb.Gas(5, 2, 3, 2)
    og = orc.gas(cp=(5, 2), cv=(3, 2))
    s_np = orc.random_state(3, 5000, seed=3)
    s = to_dev(s_np, cuda)
    assert all_same(to_host(fvb.flux(s, 3, gas=g)), orc.flux(3, s_np, gas=og))
    j, lam = fvb.jacobian(s, 3, gas=g)
    j_np, lam_np = orc.jacobian(3, s_np, gas=og)
    assert all_same(to_host(j), j_np) and lam.item() == lam_np


# ---- known answers on the device ----------------------------------------------


def test_worked_instance(cuda):
    s = [torch.tensor([v], dtype=torch.float64, device=cuda) for v in (2.0, 2.0, 4.0, 4.0, 14.0)]
    f = [t.item() for t in fvb.flux(s, 3)]
    assert [f[r * 3] for r in range(5)] == [2.0, 4.0, 4.0, 4.0, 16.0]
    c = [t.item() for t in fvb.cons2prim(s, 3)]
    assert c[:4] == [1.0, 2.0, 2.0, 2.0] and c[4] == 1.1832159566199232
    j, lam = fvb.jacobian(s, 3)
    A0 = np.array([t.item() for t in j[:25]]).reshape(5, 5)
    assert np.allclose(A0, [[0, 1, 0, 0, 0], [0.8, 1.6, -0.8, -0.8, 0.4], [-2, 2, 1, 0, 0],
                            [-2, 2, 0, 1, 0], [-6.2, 7.6, -0.8, -0.8, 1.4]], rtol=0, atol=1e-15)
    assert lam.item() == 4.183215956619923


# ---- layout edge cases ----------------------------------------------------------


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_unaligned_and_mixed_residue_planes(cuda, orc, prec):
    # Slices at element offsets exercise the scalar head/tail, and planes with
    # different 32-byte residues the element-wide fallback.
    dim, n = 3, 5003
    s_np = orc.random_state(dim, n, seed=77, prec=prec)
    want = orc.flux(dim, s_np)
    for offsets in [(1,) * 5, (3,) * 5, (0, 1, 2, 3, 1)]:
        s = []
        for a, off in zip(s_np, offsets):
            buf = torch.empty(n + 8, dtype=DT[prec], device=cuda)
            buf[off:off + n] = torch.from_numpy(a).to(cuda)
            s.append(buf[off:off + n])
        outs = []
        for j in range(15):
            buf = torch.empty(n + 8, dtype=DT[prec], device=cuda)
            off = offsets[j % 5]
            outs.append(buf[off:off + n])
        fvb.flux(s, dim, out=outs)
        assert all_same(to_host(outs), want), offsets


def test_validation_errors(cuda):
    a = torch.zeros(10, dtype=torch.float64, device=cuda)
    b = torch.zeros(11, dtype=torch.float64, device=cuda)
    c = torch.zeros(10, dtype=torch.float32, device=cuda)
    with pytest.raises(fvb.LengthMismatch):
        fvb.flux([a, a, a, a, b], 3)
    with pytest.raises(fvb.PrecisionError):
        fvb.flux([a, a, a, a, c], 3)
    with pytest.raises(fvb.ArgumentError):
        fvb.flux([a, a, a], 3)


# ---- CFL maximum ------------------------------------------------------------------


def test_lambda_max_exact_and_nan(cuda, orc):
    dim, n = 3, 2_000_003
    s_np = orc.random_state(dim, n, seed=5)
    s = to_dev(s_np, cuda)
    _, lam = fvb.wave_speed_max(s, dim)
    assert lam.item() == orc.wave_speed_max(dim, s_np)
    # NaN anywhere propagates (CFL max definition)
    s[0][n // 2] = float("nan")
    _, lam = fvb.wave_speed_max(s, dim)
    assert np.isnan(lam.item())
    # empty range -> 0
    e = [torch.empty(0, dtype=torch.float64, device=cuda) for _ in range(5)]
    _, lam = fvb.wave_speed_max(e, dim)
    assert lam.item() == 0.0


def test_lambda_max_output_is_validated(cuda, orc):
    # the caller's accumulator must be one element of the state's precision on
    # the state's device: anything else would be an out-of-bounds or foreign
    # device write (memset + atomicMax of sizeof(T) bytes)
    s = fvb.synth_state(3, 1000, prec=1)
    for bad, err in [(torch.empty((), dtype=torch.float32, device=cuda), fvb.PrecisionError),
                     (torch.empty((), dtype=torch.float64), fvb.ArgumentError),
                     (torch.empty(0, dtype=torch.float64, device=cuda), fvb.ArgumentError)]:
        with pytest.raises(err):
            fvb.jacobian(s, 3, lambda_max=bad)
        with pytest.raises(err):
            fvb.wave_speed_max(s, 3, lambda_max=bad)
    # a refused call enqueues nothing: the caller's word keeps its value
    lam = torch.full((), 7.0, dtype=torch.float64, device=cuda)
    outs = [torch.empty(1000, dtype=torch.float64, device=cuda) for _ in range(75)]
    raw = torch.empty(1001 * 8, dtype=torch.uint8, device=cuda)
    odd = raw[4:4 + 1000 * 8].view(torch.float32)  # a misaligned f64 plane, by pointer
    args = [t.data_ptr() for t in s]
    args[2] = odd.data_ptr()
    for fn, extra in [(N.lib().fvb_jacobian, [N.ptr_array([t.data_ptr() for t in outs])]),
                      (N.lib().fvb_wave_speed_max, [None])]:
        with pytest.raises(fvb.ArgumentError):
            N.check(fn(None, 3, 1, 1000, N.ptr_array(args), *extra, lam.data_ptr(),
                       torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert lam.item() == 7.0


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_cfl_lambda_max_on_a_side_stream(cuda, orc, prec):
    # shard.cfl_lambda_max with the reduction on the caller's stream: the
    # widening copy (and, under torch.distributed, the all-reduce) on the
    # current stream must wait for it; a torch stream and a raw handle
    from paper_1809_09851_b200 import shard
    dim, n = 3, 2_000_003
    s_np = orc.random_state(dim, n, seed=21, prec=prec)
    s = to_dev(s_np, cuda)
    want = float(orc.wave_speed_max(dim, s_np))
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    for st in (side, side.cuda_stream):
        with torch.cuda.stream(side):
            torch.cuda._sleep(2_000_000)  # the reduction lands late on the side stream
        lam = shard.cfl_lambda_max(s, dim, stream=st)
        assert lam.dtype == torch.float64 and lam.item() == want


def test_lambda_invariant_to_slicing(cuda, orc):
    # Shard the range like the multi-GPU path; the max over slice maxima is
    # bitwise the global max (order-independent reduction).
    dim, n = 3, 1_000_001
    s = fvb.synth_state(dim, n, seed=0x5EED)
    _, whole = fvb.wave_speed_max(s, dim)
    for G in (2, 3, 8):
        parts = []
        for g in range(G):
            lo, hi = g * n // G, (g + 1) * n // G
            _, m = fvb.wave_speed_max([t[lo:hi] for t in s], dim)
            parts.append(m.item())
        assert max(parts) == whole.item()


# ---- axpy-sin: sin within 4 ulp --------------------------------------------------


def test_axpy_sin(cuda, orc):
    z = np.load(os.path.join(GOLDEN, "axpy_sin.npz"))
    x, y = to_dev([z["x"], z["y"]], cuda)
    fvb.axpy_sin(x, y)  # in place, dest aliases a leaf
    got = y.cpu().numpy()
    assert ulp_diff(got, z["y_out"]).max() <= 4
    x32, y32 = to_dev([z["x32"], z["y32"]], cuda)
    fvb.axpy_sin(x32, y32)
    got32 = y32.cpu().numpy().astype(np.float64)
    want32 = z["y32_out"].astype(np.float64)
    assert np.all(np.abs(got32 - want32) <= 1e-6 * np.maximum(np.abs(want32), 1.0))
    # Figure 2: x=0, y=pi/2 -> 0.5
    x = torch.zeros(1, dtype=torch.float64, device=cuda)
    y = torch.full((1,), np.pi / 2, dtype=torch.float64, device=cuda)
    assert abs(fvb.axpy_sin(x, y).item() - 0.5) <= 1e-15


def test_axpy_sin_config1(cuda, orc):
    # C1 at full size: N = 1e6 from the device generator, against the oracle
    n = 1_000_000
    x = fvb.synth_uniform(n, seed=1, first=0)
    y = fvb.synth_uniform(n, seed=1, first=n)
    want = orc.axpy_sin(orc.make_vec(1, 0, n), orc.make_vec(1, n, n))
    fvb.axpy_sin(x, y)
    assert ulp_diff(y.cpu().numpy(), want).max() <= 4


# ---- full-size properties (BASELINE configs) ----------------------------------------


def test_flux_1e8_sampled_bitwise(cuda, orc):
    # C3 at N = 1e8 (16 GB of planes): every sampled point equals the oracle
    # evaluated on the same global point (random-access generator).
    dim, n = 3, 100_000_000
    s = fvb.synth_state(dim, n, seed=0x5EED)
    f = fvb.flux(s, dim)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    idx = np.unique(np.concatenate([rng.integers(0, n, 2000), [0, 1, n - 2, n - 1]]))
    it = torch.from_numpy(idx).to(cuda)
    got = np.stack([t[it].cpu().numpy() for t in f])
    for k, i in enumerate(idx):
        pt = orc.random_state(dim, 1, seed=0x5EED, first=int(i))
        want = np.array([a[0] for a in orc.flux(dim, pt)])
        assert same_bits(got[:, k], want), int(i)
    # row 0 is the momentum planes bit for bit
    for j in range(3):
        assert torch.equal(f[j].view(torch.int64), s[1 + j].view(torch.int64))
    del f, s
    torch.cuda.empty_cache()


def test_jacobian_cfl_1e8(cuda, orc):
    # C4 at N = 1e8 (f32: 32 GB of outputs): sampled bitwise, fused lambda_max
    # equals the standalone reduction and the max of per-point lambda.
    dim, n = 3, 100_000_000
    s = fvb.synth_state(dim, n, prec=0, seed=0x5EED)
    j, lam = fvb.jacobian(s, dim)
    lam_pts = torch.empty_like(s[0])
    _, lam2 = fvb.wave_speed_max(s, dim, lam_out=lam_pts)
    torch.cuda.synchronize()
    assert lam.item() == lam2.item() == lam_pts.max().item()
    rng = np.random.default_rng(1)
    idx = rng.integers(0, n, 300)
    it = torch.from_numpy(idx).to(cuda)
    got = np.stack([t[it].cpu().numpy() for t in j])
    for k, i in enumerate(idx):
        pt = orc.random_state(dim, 1, seed=0x5EED, first=int(i), prec="f32")
        want = np.array([a[0] for a in orc.jacobian(dim, pt)[0]], np.float32)
        assert same_bits(got[:, k], want), int(i)
    # size-independent property over all 1e8 points: Euler homogeneity,
    # A_k(U) U = F_k(U), against the separately computed flux,
    # accumulated in f64 from the f32 planes
    f = fvb.flux(s, dim)
    w = dim + 2
    for kk in range(dim):
        for r in range(w):
            au = torch.zeros(n, dtype=torch.float64, device=cuda)
            for c in range(w):
                au += j[(kk * w + r) * w + c].double() * s[c].double()
            fk = f[r * dim + kk].double()
            err = (au - fk).abs() / torch.clamp(fk.abs(), min=1.0)
            assert float(err.max()) < 1e-5, (kk, r, float(err.max()))
    del j, s, lam_pts, f
    torch.cuda.empty_cache()


# ---- the host-buffer (end-to-end) path -----------------------------------------------


@pytest.mark.parametrize("pinned", [True, False])
def test_host_path_matches_device(cuda, orc, pinned):
    dim, n = 3, 3_000_017
    s_np = orc.random_state(dim, n, seed=11)
    want = orc.flux(dim, s_np)
    ctx = fvb.HostContext(0, chunk_points=1 << 20)
    hs = [torch.from_numpy(a) for a in s_np]
    outs = [torch.empty(n, dtype=torch.float64) for _ in range(15)]
    if pinned:
        hs = [t.pin_memory() for t in hs]
        outs = [t.pin_memory() for t in outs]
    ctx.flux(hs, dim, outs)
    assert all_same([t.numpy() for t in outs], want)
    jo = [torch.empty(n, dtype=torch.float64) for _ in range(75)]
    _, lam = ctx.jacobian(hs, dim, jo)
    j_np, lam_np = orc.jacobian(dim, s_np)
    assert lam == lam_np
    # all 75, the 30 constant entries filled host-side included
    assert all_same([t.numpy() for t in jo], j_np)
    ctx.close()


@pytest.mark.parametrize("outputs", ["device", "reduce_only"])
def test_host_path_pageable_inputs_busy_stream(cuda, orc, outputs):
    # Pageable inputs bounce through the slot's pinned buffer; chunk c+3 is
    # packed into the buffer chunk c used.  With device (or no) outputs no
    # unpack waits on the slot, and with the `after` stream still busy every
    # H2D is queued behind it -- the packing must wait for chunk c's copies
    # anyway, else chunk c computes on chunk c+3's data.
    dim, n = 3, 1_000_003
    s_np = orc.random_state(dim, n, seed=21)
    ctx = fvb.HostContext(0, chunk_points=1 << 13)  # 123 chunks
    k = _flux_kernel() if outputs == "device" else None
    busy = torch.cuda.Stream()
    with torch.cuda.stream(busy):
        torch.cuda._sleep(400_000_000)  # ~0.2 s of queued work ahead of the pipeline
    if outputs == "device":
        leaves = [None] * k.n_inputs
        for ci in range(k.n_inputs):
            leaves[k.in_slot[ci]] = torch.from_numpy(s_np[ci])
        outs = [torch.empty(n, dtype=torch.float64, device=cuda) for _ in range(15)]
        ctx.launch(k, outs + leaves, n, after=busy)
        assert all_same([t.cpu().numpy() for t in outs], orc.flux(dim, s_np))
    else:
        import re
        import struct
        pat = dict(fvb.patterns())["wave_speed3_f64"]
        kw = fvb.lookup(re.sub(r"Cd#(\w+);", lambda m: "Cd%016x;" % struct.unpack(
            "<Q", struct.pack("<d", {"half": 0.5, "gm1": 0.4, "gamma": 1.4}[m.group(1)]))[0],
            pat))
        lv = [None] * kw.n_inputs
        for ci in range(kw.n_inputs):
            lv[kw.in_slot[ci]] = torch.from_numpy(s_np[ci])
        lam = ctx.launch(kw, [None] + lv, n, reduce=True, after=busy)
        assert lam == orc.wave_speed_max(dim, s_np)
    ctx.close()


def test_host_path_rejects_one_plane_for_two_outputs(cuda, orc):
    # host threads write the pass-through / constant outputs while the
    # pipeline writes the rest: one plane named twice would race
    s_np = orc.random_state(3, 1000, seed=3)
    hs = [torch.from_numpy(a) for a in s_np]
    ctx = fvb.HostContext(0)
    outs = [torch.empty(1000, dtype=torch.float64) for _ in range(75)]
    outs[40] = outs[7]
    with pytest.raises(fvb.ArgumentError):
        ctx.jacobian(hs, 3, outs)
    fo = [torch.empty(1000, dtype=torch.float64) for _ in range(15)]
    fo[0] = fo[9]
    with pytest.raises(fvb.ArgumentError):
        ctx.flux(hs, 3, fo)
    ctx.close()


def test_host_path_refuses_device_planes_before_host_threads(cuda, orc):
    # the raw C ABI handed device pointers as host planes: refused with
    # FVB_EARG before any host thread touches them (the pass-through rows,
    # the Jacobian's constant fills), not a wild host access
    n = 4096
    s = [t for t in fvb.synth_state(3, n, prec=1)]
    ctx = fvb.HostContext(0)
    hs = [torch.empty(n, dtype=torch.float64) for _ in range(5)]
    for ins, outs, count in (
        (s, [torch.empty(n, dtype=torch.float64) for _ in range(15)], 15),       # device inputs
        (hs, [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(15)], 15),
    ):
        st = N.lib().fvb_flux_host(ctx._h, None, 3, 1, n, N.ptr_array([t.data_ptr() for t in ins]),
                                   N.ptr_array([t.data_ptr() for t in outs]))
        assert st == N.FVB_EARG and b"device memory" in N.lib().fvb_last_error()
    jo = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(75)]
    lam = ctypes.c_double()
    st = N.lib().fvb_jacobian_host(ctx._h, None, 3, 1, n, N.ptr_array([t.data_ptr() for t in hs]),
                                   N.ptr_array([t.data_ptr() for t in jo]), ctypes.byref(lam))
    assert st == N.FVB_EARG and b"device memory" in N.lib().fvb_last_error()
    # fvb_launch_host: a device plane flagged as host (arg_on_device 0)
    import re
    import struct
    pat = dict(fvb.patterns())["pressure3_f64"]
    kp = fvb.lookup(re.sub(r"Cd#(\w+);", lambda m: "Cd%016x;" % struct.unpack(
        "<Q", struct.pack("<d", {"half": 0.5, "gm1": 0.4}[m.group(1)]))[0], pat))
    count = 1 + kp.n_inputs
    for ptrs in ([jo[0].data_ptr()] + [t.data_ptr() for t in hs[:kp.n_inputs]],
                 [hs[0].data_ptr()] + [t.data_ptr() for t in s[:kp.n_inputs]]):
        st = N.lib().fvb_launch_host(ctx._h, ctypes.byref(kp), n, N.ptr_array(ptrs),
                                     (ctypes.c_uint8 * count)(*([1] * count)),
                                     (ctypes.c_uint8 * count)(*([0] * count)), None, None)
        assert st == N.FVB_EARG and b"device memory" in N.lib().fvb_last_error()
    # a host plane that is not element-aligned (host threads fill and copy
    # element-wise): refused with FVB_EALIGN
    raw = torch.empty(n * 8 + 8, dtype=torch.uint8)
    odd = raw.data_ptr() + 4
    outs = [torch.empty(n, dtype=torch.float64) for _ in range(15)]
    ptrs = [t.data_ptr() for t in outs]
    ptrs[3] = odd
    st = N.lib().fvb_flux_host(ctx._h, None, 3, 1, n, N.ptr_array([t.data_ptr() for t in hs]),
                               N.ptr_array(ptrs))
    assert st == N.FVB_EALIGN
    # the context still works afterwards
    s_np = orc.random_state(3, n, seed=11)
    fo = [torch.empty(n, dtype=torch.float64) for _ in range(15)]
    ctx.flux([torch.from_numpy(a) for a in s_np], 3, fo)
    assert all(a.numpy().tobytes() == b.tobytes() for a, b in zip(fo, orc.flux(3, s_np)))
    ctx.close()


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_host_jacobian_constant_fills(cuda, orc, prec):
    # the constant entries (0, 1, gamma-1) are filled by host threads: every
    # dimension, both precisions, a non-default gas (another gamma-1), and
    # outputs pre-filled with garbage so a skipped fill would show
    g, og = fvb.Gas(5, 2, 3, 2), orc.gas(cp=(5, 2), cv=(3, 2))
    ctx = fvb.HostContext(0, chunk_points=1 << 12)
    for dim in (1, 2, 3):
        s_np = orc.random_state(dim, 20_011, seed=31 + dim, prec=prec)
        hs = [torch.from_numpy(a) for a in s_np]
        jo = [torch.full((20_011,), float("nan"), dtype=DT[prec]) for _ in range(dim * (dim + 2) ** 2)]
        _, lam = ctx.jacobian(hs, dim, jo, gas=g)
        j_np, lam_np = orc.jacobian(dim, s_np, gas=og)
        assert lam == lam_np
        assert all_same([t.numpy() for t in jo], j_np), dim
    ctx.close()


def _flux_kernel():
    import re
    import struct
    pat = dict(fvb.patterns())["flux3_f64"]
    return fvb.lookup(re.sub(r"Cd#(\w+);", lambda m: "Cd%016x;" % struct.unpack(
        "<Q", struct.pack("<d", {"half": 0.5, "gm1": 0.4}[m.group(1)]))[0], pat))


@pytest.mark.parametrize("mode", ["pageable", "pinned", "mixed"])
def test_launch_host_any_kernel(cuda, orc, mode):
    # fvb_launch_host: a structural-key kernel over host arrays -- pageable
    # (bounced through pinned buffers by the copy threads), pinned (DMA'd
    # directly) or a mix with device-resident leaves and device outputs --
    # over several chunks; bitwise the oracle.
    dim, n = 3, 1_000_003
    s_np = orc.random_state(dim, n, seed=13)
    want = orc.flux(dim, s_np)
    k = _flux_kernel()
    ctx = fvb.HostContext(0, chunk_points=1 << 18)
    leaves = [None] * k.n_inputs
    for ci in range(k.n_inputs):
        leaves[k.in_slot[ci]] = torch.from_numpy(s_np[ci])
    outs = [torch.empty(n, dtype=torch.float64) for _ in range(15)]
    on_dev = [0] * (15 + k.n_inputs)
    if mode == "pinned":
        leaves = [t.pin_memory() for t in leaves]
        outs = [t.pin_memory() for t in outs]
    elif mode == "mixed":
        for i in (0, 2):
            leaves[i] = leaves[i].to(cuda)
            on_dev[15 + i] = 1
        for j in (1, 7):
            outs[j] = torch.empty(n, dtype=torch.float64, device=cuda)
            on_dev[j] = 1
    args = N.ptr_array([t.data_ptr() for t in outs + leaves])
    prec = (ctypes.c_uint8 * len(on_dev))(*([1] * len(on_dev)))
    dev = (ctypes.c_uint8 * len(on_dev))(*on_dev)
    N.check(N.lib().fvb_launch_host(ctx._h, ctypes.byref(k), n, args, prec, dev, None, None))
    assert all_same([t.cpu().numpy() for t in outs], want)
    # in place: pressure written over its own (pageable) rhoE leaf
    import re
    import struct
    pat = dict(fvb.patterns())["pressure3_f64"]
    kp = fvb.lookup(re.sub(r"Cd#(\w+);", lambda m: "Cd%016x;" % struct.unpack(
        "<Q", struct.pack("<d", {"half": 0.5, "gm1": 0.4}[m.group(1)]))[0], pat))
    hs = [torch.from_numpy(a.copy()) for a in s_np]
    lv = [None] * kp.n_inputs
    for ci in range(kp.n_inputs):
        lv[kp.in_slot[ci]] = hs[ci]
    args = N.ptr_array([hs[4].data_ptr()] + [t.data_ptr() for t in lv])
    prec = (ctypes.c_uint8 * (1 + kp.n_inputs))(*([1] * (1 + kp.n_inputs)))
    N.check(N.lib().fvb_launch_host(ctx._h, ctypes.byref(kp), n, args, prec, None, None, None))
    assert same_bits(hs[4].numpy(), orc.cons2prim(dim, s_np)[dim])
    # the CFL reduction with a NULL output slot (reduce only), host leaves
    pat = dict(fvb.patterns())["wave_speed3_f64"]
    kw = fvb.lookup(re.sub(r"Cd#(\w+);", lambda m: "Cd%016x;" % struct.unpack(
        "<Q", struct.pack("<d", {"half": 0.5, "gm1": 0.4, "gamma": 1.4}[m.group(1)]))[0], pat))
    lv = [None] * kw.n_inputs
    for ci in range(kw.n_inputs):
        lv[kw.in_slot[ci]] = torch.from_numpy(s_np[ci])
    # (through the HostContext.launch wrapper; a None plane is a NULL slot)
    assert ctx.launch(kw, [None] + lv, n, reduce=True) == orc.wave_speed_max(dim, s_np)
    # overlapping host planes at an offset are refused
    buf = torch.empty(n + 8, dtype=torch.float64)
    bad = [buf[:n], buf[3:n + 3]] + [torch.empty(n, dtype=torch.float64) for _ in range(13)]
    args = N.ptr_array([t.data_ptr() for t in bad + [torch.from_numpy(a) for a in s_np]])
    prec = (ctypes.c_uint8 * 20)(*([1] * 20))
    with pytest.raises(fvb.ArgumentError):
        N.check(N.lib().fvb_launch_host(ctx._h, ctypes.byref(k), n, args, prec, None, None,
                                        None))
    ctx.close()


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("pinned", [False, True])
def test_launch_host_jacobian_host_side_writes(cuda, orc, prec, pinned):
    # fvb_launch_host with the hand-written Jacobian kernel (the reference's
    # Jacobian block through the adapter or the JIT seam): its constant
    # entries are filled and its duplicate entries copied host-side.  Outputs
    # start as NaN, so a skipped host-side write shows; a non-default gas
    # (another gamma-1), d = 2 and 3, a CFL reduction, several chunks; one
    # output on the device and one output slot aliasing nothing special.
    import re
    import struct
    g, og = fvb.Gas(5, 2, 3, 2), orc.gas(cp=(5, 2), cv=(3, 2))
    consts = {"half": 0.5, "gm1": g.gamma_minus_one, "gamma": g.gamma, "zero": 0.0, "one": 1.0}
    c = "d" if prec == "f64" else "s"
    ctx = fvb.HostContext(0, chunk_points=1 << 14)
    for dim in (2, 3):
        n = 100_003
        k = fvb.lookup(re.sub(r"C([sd])#(\w+);", lambda m: "C%s%016x;" % (m.group(1), struct.unpack(
            "<Q", struct.pack("<d", consts[m.group(2)]))[0]),
            dict(fvb.patterns())[f"jacobian{dim}_{prec}"]))
        assert k.name.decode().startswith("jacobian")
        s_np = orc.random_state(dim, n, seed=40 + dim, prec=prec)
        want, lam_w = orc.jacobian(dim, s_np, gas=og)
        leaves = [None] * k.n_inputs
        for ci in range(k.n_inputs):
            leaves[k.in_slot[ci]] = torch.from_numpy(s_np[ci])
        outs = [torch.full((n,), float("nan"), dtype=DT[prec]) for _ in range(k.n_outputs)]
        if pinned:
            leaves = [t.pin_memory() for t in leaves]
            outs = [t.pin_memory() for t in outs]
        outs[1] = outs[1].to(cuda)  # row 0, column 1 (a constant entry) on the device
        lam = ctx.launch(k, outs + leaves, n, reduce=True)
        assert lam == lam_w, dim
        assert all_same([t.cpu().numpy() for t in outs], want), (dim, c)
    ctx.close()


# ---- structural-key kernels -----------------------------------------------------------


def test_lookup_kernel_launch(cuda, orc):
    import re
    import struct

    def hexbits(v):
        return "%016x" % struct.unpack("<Q", struct.pack("<d", v))[0]

    pat = dict(fvb.patterns())["flux3_f64"]
    key = re.sub(r"Cd#(\w+);", lambda m: "Cd" + hexbits({"half": 0.5, "gm1": 0.4}[m.group(1)])
                 + ";", pat)
    k = fvb.lookup(key)
    n = 10_007
    s_np = orc.random_state(3, n, seed=21)
    s = to_dev(s_np, cuda)
    names = ["rho", "m0", "m1", "m2", "E"]
    # argument block: 15 outputs, then leaves in the key's slot order
    slots = [None] * k.n_inputs
    for ci in range(5):
        slots[k.in_slot[ci]] = s[ci]
    outs = [torch.empty(n, dtype=torch.float64, device=cuda) for _ in range(15)]
    args = N.ptr_array([t.data_ptr() for t in outs + slots])
    # two halves through [begin, end), like JitKernel::Fn ranges
    stream = torch.cuda.current_stream().cuda_stream
    for b, e in ((0, 5000), (5000, n)):
        N.check(k.fn(ctypes.byref(k), b, e, args, stream))
    assert all_same(to_host(outs), orc.flux(3, s_np))
    assert names  # canonical order documented in fvb_registry.cu


def test_in_place_rules(cuda, orc):
    import re
    import struct

    dim, n = 3, 4099
    s_np = orc.random_state(dim, n, seed=31)
    want = orc.flux(dim, s_np)
    s = to_dev(s_np, cuda)
    outs = [torch.empty(n, dtype=torch.float64, device=cuda) for _ in range(15)]
    # the direct entry points reject an output that is an input plane ...
    bad = list(outs)
    bad[3] = s[1]
    with pytest.raises(fvb.ArgumentError):
        fvb.flux(s, dim, out=bad)
    # ... and partially overlapping planes, before any launch
    buf = torch.empty(2 * n, dtype=torch.float64, device=cuda)
    bad = list(outs)
    bad[0], bad[1] = buf[:n], buf[5:n + 5]
    with pytest.raises(fvb.ArgumentError):
        fvb.flux(s, dim, out=bad)
    # one plane named by two outputs holds the later item (the reference's
    # item order)
    dup = list(outs)
    dup[1] = dup[0]
    fvb.flux(s, dim, out=dup)
    assert same_bits(to_host([dup[0]])[0], want[1])
    # structural-key kernels evaluate in place, as JitKernel::Fn may:
    # pressure written over its own rhoE leaf equals the oracle bit for bit
    vals = {"half": 0.5, "gm1": 0.4}
    pat = dict(fvb.patterns())["pressure3_f64"]
    k = fvb.lookup(re.sub(r"Cd#(\w+);", lambda m: "Cd%016x;" % struct.unpack(
        "<Q", struct.pack("<d", vals[m.group(1)]))[0], pat))
    assert k.n_outputs == 1
    slots = [None] * k.n_inputs
    for ci in range(k.n_inputs):
        slots[k.in_slot[ci]] = s[ci]
    args = N.ptr_array([s[4].data_ptr()] + [t.data_ptr() for t in slots])
    N.check(k.fn(ctypes.byref(k), 0, n, args, torch.cuda.current_stream().cuda_stream))
    assert same_bits(to_host([s[4]])[0], orc.cons2prim(dim, s_np)[dim])


def test_cuda_graph_capture(cuda, orc):
    dim, n = 3, 100_000
    s = fvb.synth_state(dim, n, seed=9)
    out = [torch.empty(n, dtype=torch.float64, device=cuda) for _ in range(15)]
    g = torch.cuda.CUDAGraph()
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        fvb.flux(s, dim, out=out)  # warm (occupancy query) outside capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=stream):
            fvb.flux(s, dim, out=out)
    for t in out:
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    want = orc.flux(dim, [t.cpu().numpy() for t in s])
    assert all_same(to_host(out), want)


# ---- IEEE special values -----------------------------------------------------------


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_special_values(cuda, orc, prec, dim):
    # zero / negative density, +-0, +-inf, NaN, the smallest denormal:
    # bitwise except NaN payloads (both NaN suffices), like the oracle vs the
    # reference (test_oracle.py::test_special_values_vs_reference)
    from tests.test_oracle import nan_aware_equal, special_state
    s_np = special_state(dim, prec)
    s = to_dev(s_np, cuda)
    for got, want in [(fvb.flux(s, dim), orc.flux(dim, s_np)),
                      (fvb.cons2prim(s, dim), orc.cons2prim(dim, s_np)),
                      (fvb.jacobian(s, dim)[0], orc.jacobian(dim, s_np)[0])]:
        got = to_host(got)
        assert all(nan_aware_equal(x, y) for x, y in zip(got, want))
    _, lam = fvb.wave_speed_max(s, dim)
    assert np.isnan(lam.item())


def test_cons2prim_1e8_sampled_and_round_trip(cuda, orc):
    # C2 at N = 1e8: sampled points bitwise against the oracle at the same
    # global points; over all 1e8 points the size-independent property
    # prim2cons(cons2prim(U)) == U within 1e-12 (acceptance.cpp:244-284).
    dim, n = 1, 100_000_000
    s = fvb.synth_state(dim, n, seed=0x5EED)
    c = fvb.cons2prim(s, dim)
    back = fvb.prim2cons([s[0], c[0], c[1]], dim)
    torch.cuda.synchronize()
    for a, b in zip(back, s[1:]):
        scale = torch.clamp(torch.maximum(a.abs(), b.abs()), min=1.0)
        assert bool(((a - b).abs() <= 1e-12 * scale).all())
    rng = np.random.default_rng(2)
    idx = np.unique(np.concatenate([rng.integers(0, n, 2000), [0, n - 1]]))
    it = torch.from_numpy(idx).to(cuda)
    got = np.stack([t[it].cpu().numpy() for t in c])
    for k, i in enumerate(idx):
        pt = orc.random_state(dim, 1, seed=0x5EED, first=int(i))
        want = np.array([a[0] for a in orc.cons2prim(dim, pt)])
        assert same_bits(got[:, k], want), int(i)
    del s, c, back
    torch.cuda.empty_cache()


def test_beyond_32bit_indices(cuda, orc):
    # Maximum sizes: 2^32 + 4099 points (f32 d=1, 69 GB of planes), so element
    # indices, vector groups and the generator's global index all pass 2^32.
    # Points sampled around 2^31 and 2^32 and at the end equal the oracle bit
    # for bit, and the fused maximum is the max over every per-point lambda.
    dim, n = 1, (1 << 32) + 4099
    need = 4 * n * 4 + (2 << 30)
    if torch.cuda.mem_get_info()[0] < need:
        pytest.skip("needs ~71 GB of free device memory")
    s = fvb.synth_state(dim, n, prec=0, seed=0x5EED)
    lam_pts = torch.empty_like(s[0])
    _, lam = fvb.wave_speed_max(s, dim, lam_out=lam_pts)
    torch.cuda.synchronize()
    assert lam.item() == lam_pts.max().item()
    idx = np.unique(np.concatenate([
        np.arange(0, 64), np.arange((1 << 31) - 64, (1 << 31) + 64),
        np.arange((1 << 32) - 64, (1 << 32) + 64), np.arange(n - 64, n),
        np.random.default_rng(3).integers(0, n, 200)]))
    it = torch.from_numpy(idx).to(cuda)
    got_state = np.stack([t[it].cpu().numpy() for t in s])
    got_lam = lam_pts[it].cpu().numpy()
    for k, i in enumerate(idx):
        pt = orc.random_state(dim, 1, seed=0x5EED, first=int(i), prec="f32")
        assert same_bits(got_state[:, k], np.array([a[0] for a in pt], np.float32)), int(i)
        assert np.float32(orc.wave_speed_max(dim, pt)).tobytes() == got_lam[k].tobytes(), int(i)
    del s, lam_pts
    torch.cuda.empty_cache()


# ---- CSR block matvec ------------------------------------------------


def _csr_to_dev(rp, ci, v, cuda):
    return (torch.from_numpy(rp.view(np.int64)).to(cuda),
            torch.from_numpy(ci.view(np.int64)).to(cuda), torch.from_numpy(v).to(cuda))


def stencil7(n):
    """7-point Laplacian on an n^3 grid, rows column-sorted (as stored)."""
    rows = n ** 3
    r = np.arange(rows, dtype=np.int64)
    i, j, k = r % n, (r // n) % n, r // (n * n)
    offs = [-(n * n), -n, -1, 0, 1, n, n * n]
    ok = [k > 0, j > 0, i > 0, np.ones(rows, bool), i + 1 < n, j + 1 < n, k + 1 < n]
    cols = np.stack([r + o for o in offs], 1)
    mask = np.stack(ok, 1)
    vals = np.where(np.arange(7) == 3, 6.0, -1.0)[None, :].repeat(rows, 0)
    counts = mask.sum(1)
    rp = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    return rp, cols[mask].astype(np.uint64), vals[mask].astype(np.float64)


@pytest.fixture(params=["auto", "row", "warp", "pipe"])
def csr_mode(request, monkeypatch):
    # the library reads FVB_CSR_MODE per call
    if request.param != "auto":
        monkeypatch.setenv("FVB_CSR_MODE", request.param)
    return request.param


@pytest.mark.parametrize("idx", ["u64", "u32"])
@pytest.mark.parametrize("y_prec,x_prec", [("f64", "f64"), ("f64", "f32"), ("f32", "f64"),
                                           ("f32", "f32")])
def test_csr_matvec_bitwise(cuda, orc, y_prec, x_prec, csr_mode, idx):
    # Every CSR form against the oracle (pinned to the reference in
    # test_oracle.py): rows longer than one staging tile, warps whose range
    # spans several tiles, empty rows,
    # a ragged last warp / block, 7-point stencils -- and the accumulation
    # into a nonzero y.
    from tests.test_oracle import random_csr
    rng = np.random.default_rng(11)
    yt = {"f64": np.float64, "f32": np.float32}
    cases = [random_csr(rng, 1, 1, 1), random_csr(rng, 37, 3000, 1000, 3),
             random_csr(rng, 4099, 5000, 40, 9), random_csr(rng, 3001, 900, 9, 5),
             stencil7(48), stencil7(7)]
    for rp, ci, v in cases:
        rows = len(rp) - 1
        cols = int(ci.max()) + 1 if len(ci) else 1
        x = rng.uniform(-2, 2, cols).astype(yt[x_prec])
        y0 = rng.uniform(-1, 1, rows).astype(yt[y_prec])
        want = orc.csr_matvec_acc(rp, ci, v, x, y0)
        drp, dci, dv = _csr_to_dev(rp, ci, v, cuda)
        if idx == "u32":  # the narrow device layout (fvb_csr_matvec_acc_u32)
            dci = dci.to(torch.int32)
        dx = torch.from_numpy(x).to(cuda)
        dy = torch.from_numpy(y0.copy()).to(cuda)
        fvb.csr_matvec_acc(drp, dci, dv, dx, dy)
        assert same_bits(to_host([dy])[0], want), rows


@pytest.mark.parametrize("v_off,c_off", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_csr_matvec_odd_plane_offsets(cuda, orc, v_off, c_off, csr_mode):
    # values / column indices starting 8 bytes past a 16-byte boundary
    # (offset planes a caller may pass through the C ABI)
    rng = np.random.default_rng(12)
    for rp, ci, v in (stencil7(33), stencil7(5)):
        rows = len(rp) - 1
        x = rng.uniform(-2, 2, rows)
        y0 = rng.uniform(-1, 1, rows)
        want = orc.csr_matvec_acc(rp, ci, v, x, y0)
        dv = torch.from_numpy(np.concatenate([[np.nan] * v_off, v])).to(cuda)[v_off:]
        dci = torch.from_numpy(np.concatenate([[2 ** 62] * c_off, ci.view(np.int64)])
                               .astype(np.int64)).to(cuda)[c_off:]
        drp = torch.from_numpy(rp.view(np.int64)).to(cuda)
        assert (dv.data_ptr() % 16 == 8) == bool(v_off) and (dci.data_ptr() % 16 == 8) == bool(c_off)
        dy = torch.from_numpy(y0.copy()).to(cuda)
        fvb.csr_matvec_acc(drp, dci, dv, torch.from_numpy(x).to(cuda), dy)
        assert same_bits(to_host([dy])[0], want), (rows, v_off, c_off)


def test_host_path_without_bounce_buffers(cuda):
    # With no pinned memory to spare (forced here by FVB_HOST_BOUNCE=0) the
    # pageable host path falls back to plain cudaMemcpyAsync: still bitwise.
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, oracle, paper_1809_09851_b200 as fvb
orc = oracle.oracle()
s = orc.random_state(3, 300_001, seed=17)
ctx = fvb.HostContext(0, chunk_points=1 << 16)
out = [torch.empty(300_001, dtype=torch.float64) for _ in range(15)]
ctx.flux([torch.from_numpy(a) for a in s], 3, out)
want = orc.flux(3, s)
assert all(o.numpy().tobytes() == w.tobytes() for o, w in zip(out, want))
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FVB_HOST_BOUNCE="0")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_eos_bitwise(cuda, orc, prec):
    # fvb_eos against the oracle (pinned to the reference in test_oracle.py),
    # default and monatomic gas, ragged n; either output may be NULL
    rng = np.random.default_rng(6)
    for n in (1, 7, 4099, 1_000_003):
        rho = rng.uniform(0.1, 5.0, n).astype(NP[prec])
        e = rng.uniform(0.1, 9.0, n).astype(NP[prec])
        for gas, g in [(None, orc.gas()), (fvb.Gas(5, 2, 3, 2), orc.gas((5, 2), (3, 2)))]:
            p, T = fvb.eos(*to_dev([rho, e], cuda), gas=gas)
            want_p, want_T = orc.eos(rho, e, gas=g)
            assert all_same(to_host([p, T]), [want_p, want_T]), n
    d_rho, d_e = to_dev([rho, e], cuda)
    T_only = torch.empty_like(d_rho)
    N.check(N.lib().fvb_eos(None, PREC[prec], n, d_rho.data_ptr(), d_e.data_ptr(), None,
                            T_only.data_ptr(), torch.cuda.current_stream().cuda_stream))
    assert same_bits(to_host([T_only])[0], orc.eos(rho, e)[1])


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_many_gases_bitwise(cuda, orc, prec):
    # the device blocks under the gases test_oracle.py pins to the reference
    from tests.test_oracle import RANDOM_GASES
    for cp, cv in RANDOM_GASES:
        g = fvb.Gas(cp[0], cp[1], cv[0], cv[1])
        og = orc.gas(cp=cp, cv=cv)
        for dim in (1, 2, 3):
            s_np = orc.random_state(dim, 4099, seed=sum(cp) + dim, prec=prec)
            s = to_dev(s_np, cuda)
            assert all_same(to_host(fvb.flux(s, dim, gas=g)), orc.flux(dim, s_np, gas=og))
            assert all_same(to_host(fvb.cons2prim(s, dim, gas=g)),
                            orc.cons2prim(dim, s_np, gas=og))
            j, lam = fvb.jacobian(s, dim, gas=g)
            j_np, lam_np = orc.jacobian(dim, s_np, gas=og)
            assert all_same(to_host(j), j_np), (cp, cv, dim)
            assert same_bits(lam.cpu().numpy(), np.asarray(lam_np, NP[prec]))
