#!/usr/bin/env python3
"""Benchmark: fused 3-D Euler inviscid flux on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fvb|reference]
                    [--config flux3d|cons2prim1d|jacobian3d|axpy] [--prec f64|f32]
                    [--n POINTS_PER_GPU]

One step = one pass of the hot path over one batch: the fused flux kernel over
N = 1e8 points per GPU (C3: 3-D, fp64, 5 input planes -> 15 output planes,
160 algorithmic bytes/point), inputs synthesised on the device by the
random-access SplitMix64 generator (bit-identical to the reference's host
generator) and resident in HBM before the clock starts.  Multi-GPU: one
process per GPU (torchrun), each owning the contiguous global slice
[r*N, (r+1)*N) -- weak scaling, no collective on the flux path (C4 adds the
one NCCL allreduce-max of the CFL wave speed).  Timing: CUDA events on the
launching stream, barrier + synchronize on both sides, max over ranks.

`value` is whole-job points/s with inputs resident; `e2e` is the same metric
through the host-buffer C-ABI call (fvb_flux_host) from pinned host memory,
copies included; `cpu_baseline` is the unmodified reference (oracle/_ref) on
this box's host cores.  `--impl reference` times that reference alone.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3D Euler flux Gpoints/s and HBM GB/s vs peak at 1/2/4/8 B200 vs CPU ref"
L2_BYTES = 126 * 1000 * 1000  # B200 L2 (126 MB); smaller working sets get flushed between steps

# Algorithmic bytes per point (read + write) and planes.
CONFIGS = {
    # name: (dim, n_in, n_out, default N per GPU, description)
    "flux3d": (3, 5, 15, 100_000_000, "C3: 3D Euler inviscid fluxes, all 3 directions"),
    "cons2prim1d": (1, 3, 3, 100_000_000, "C2: 1D cons->prim + ideal-gas p + sound speed"),
    "jacobian3d": (3, 5, 75, 100_000_000, "C4: 3D 5x5 flux Jacobians x3 + CFL max allreduce"),
    "axpy": (0, 2, 1, 1_000_000, "C1: UETLI y = 0.5*sin(x+y)"),
    "vmag2": (3, 4, 1, 100_000_000,
              "paper micro-benchmark (mx^2+my^2+mz^2)/rho^2 = derived_v_mag2, 3D"),
    # the remaining entry points of SURVEY §8a, same N (not BASELINE configs)
    "prim2cons3d": (3, 5, 4, 100_000_000, "3D prim->cons: m = rho*v, rhoE (rho passed through)"),
    "flux_prim3d": (3, 5, 15, 100_000_000, "3D inviscid fluxes of a primitive state"),
    "eos": (0, 2, 2, 100_000_000, "ideal-gas EOS p(rho, e), T(rho, e)"),
    "cfl3d": (3, 5, 0, 100_000_000, "3D standalone CFL max wave speed (reduction only)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fvb", choices=["fvb", "reference"])
    ap.add_argument("--config", default="flux3d", choices=sorted(CONFIGS))
    ap.add_argument("--prec", default="f64", choices=["f64", "f32"])
    ap.add_argument("--n", "--points", dest="n", type=int, default=0,
                    help="points per GPU (default: the config's)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-points", type=int, default=0,
                    help="points per rank for e2e (0: all at N=1, 2.5e7 at N>1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--l2-warm", action="store_true",
                    help="replay the K steps as one CUDA graph without L2 flushes "
                         "(time-stepping loop on an L2-resident working set; labelled)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=10_000_000,
                    help="points per reference step (bounded CPU sample)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="CPU work the cpu_baseline leg aims for (reps of the sample)")
    ap.add_argument("--out", default="", help="also append the JSON line to this file")
    a = ap.parse_args()
    if a.warmup < 3:
        ap.error("--warmup must be >= 3")
    return a


# ---- environment --------------------------------------------------------------------


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def profiled_traffic(config, prec, n):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
    from the committed `ncu --set full` capture of this kernel, scaled from
    the captured launch's points to n; None when no capture is committed."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)[f"{config}_{prec}"]
        return t["dram_bytes"] / t["points"] * n
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        "sw_power_cap": 0x4,
        "hw_slowdown": 0x8,
        "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40,
        "hw_power_brake": 0x80,
    }

    def __init__(self, index):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---- the reference arm (CPU) -----------------------------------------------------------

REF_WHICH = {"flux3d": 0, "cons2prim1d": 1, "jacobian3d": 2, "axpy": 3, "vmag2": 4,
             "prim2cons3d": 5, "flux_prim3d": 6, "eos": 7, "cfl3d": 8}


def reference_run(cfg_name, prec, steps, warmup, sample, threads):
    """Time the unmodified reference (oracle/_ref) on the host cores."""
    import oracle

    R = oracle.reference()
    if R is None:
        raise RuntimeError("oracle/_ref/libfvref.so missing (build() on a box with "
                           "/root/reference)")
    dim = CONFIGS[cfg_name][0]
    times = R.time_config(REF_WHICH[cfg_name], max(dim, 1), prec, sample, threads,
                          warmup + steps)
    t = times[warmup:]
    return sample, t


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---- the device arm -----------------------------------------------------------------------


def end_to_end(a, fvb, ins, n, n_in, n_out, dim, dt, esize, local, dist, world, dev, torch):
    """Same metric through the host-buffer C-ABI call (fvb_flux_host /
    fvb_jacobian_host / fvb_launch_host): inputs copied from pinned host memory and every
    computed output plane copied back, all inside the timed region.  The
    flux's row 0 (bit-for-bit the momentum inputs) is copied host-side by the
    library instead of crossing PCIe; it is counted separately.

    Host memory: one rank pins (n_in + n_out) planes.  With several ranks per
    box each streams a bounded slice (--e2e-points, default 2.5e7 points per
    rank when N > 1) -- the pipeline's rate is flat in the point count far
    below that -- so 8 ranks never pin more than ~32 GB between them."""
    if world > 1 and a.e2e_points == 0:
        n = min(n, 25_000_000)
    elif a.e2e_points:
        n = min(n, a.e2e_points)
    torch.cuda.empty_cache()
    host_in = torch.empty((n_in, n), dtype=dt).pin_memory()
    for i, t in enumerate(ins[:n_in]):  # (v_mag2 reads rho and m only)
        host_in[i].copy_(t[:n])
    host_in = list(host_in.unbind(0))
    host_out = list(torch.empty((n_out, n), dtype=dt).pin_memory().unbind(0))
    ctx = fvb.HostContext(local)
    kernel = planes = None
    if a.config in LAUNCH_HOST_PATTERN:
        # blocks without a named host-buffer call: the registry kernel of the
        # reference's tree through fvb_launch_host (argument block: outputs,
        # then the leaves in slot order)
        kernel = fvb.lookup(registry_key(fvb, LAUNCH_HOST_PATTERN[a.config] + "_" + a.prec))
        assert kernel.n_outputs == n_out and kernel.n_inputs == n_in, a.config
        slots = [None] * n_in
        for i in range(n_in):
            slots[kernel.in_slot[i]] = host_in[i]
        planes = host_out + slots

    def e2e_step():
        if a.config == "flux3d":
            ctx.flux(host_in, dim, host_out)
        elif a.config == "jacobian3d":
            ctx.jacobian(host_in, dim, host_out)
        else:
            ctx.launch(kernel, planes, n)

    e2e_step()  # warm (staging allocation)
    if dist is not None:
        dist.barrier()
    t_start = time.perf_counter()
    for _ in range(a.e2e_steps):
        e2e_step()  # returns after the last D2H copy completed
    e2e_s = (time.perf_counter() - t_start) / a.e2e_steps
    if dist is not None:
        te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = te.item()
    ctx.close()
    # planes written host-side instead of crossing PCIe: the flux's row 0
    # (copies of the momentum inputs), the Jacobian's constant entries
    # (JacobianOp::constant_item: 4 / 12 / 30 of 9 / 32 / 75 in 1-/2-/3-D)
    # and its duplicate entries (JacobianOp::duplicate_of: 0 / 4 / 18), copied
    # host-side from the shipped copy
    passthrough = dim if a.config == "flux3d" else 0
    filled = {1: 4, 2: 12, 3: 30}[dim] if a.config == "jacobian3d" else 0
    dups = {1: 0, 2: 4, 3: 18}[dim] if a.config == "jacobian3d" else 0
    return {"value": world * n / e2e_s / 1e9, "unit": "Gpoints/s",
            "h2d_bytes_per_step": world * n * n_in * esize,
            "d2h_bytes_per_step": world * n * (n_out - passthrough - filled - dups) * esize
                                  + (8 if a.config == "jacobian3d" else 0),
            "host_passthrough_bytes_per_step": world * n * (passthrough + dups) * esize,
            "host_fill_bytes_per_step": world * n * filled * esize,
            "ms_per_step": e2e_s * 1e3, "host_memory": "pinned", "steps": a.e2e_steps,
            "points_per_rank": n,
            "path": {"flux3d": "fvb_flux_host", "jacobian3d": "fvb_jacobian_host"}.get(
                a.config, "fvb_launch_host")}


# configs whose e2e runs the registry kernel through fvb_launch_host
LAUNCH_HOST_PATTERN = {"cons2prim1d": "cons2prim_c1", "vmag2": "v_mag23",
                       "prim2cons3d": "prim2cons3", "flux_prim3d": "flux_prim3"}
# the default gas's named constants (EosSpec(): gamma = 7/5, R = 1, cv = 5/2)
_GAS_CONSTS = {"half": 0.5, "gm1": 0.4, "gamma": 1.4, "zero": 0.0, "one": 1.0, "cv": 2.5}


def registry_key(fvb, name):
    """The structural key of registry pattern `name` with the default gas's
    constants filled in (the key the reference renders for its own tree:
    C<p><16 hex digits of the double>;)."""
    import re
    import struct
    pat = dict(fvb.patterns())[name]
    return re.sub(r"C([sd])#(\w+);",
                  lambda m: "C%s%016x;" % (m.group(1), struct.unpack(
                      "<Q", struct.pack("<d", _GAS_CONSTS[m.group(2)]))[0]), pat)



def device_run(a, rank, world, local):
    import torch

    import paper_1809_09851_b200 as fvb
    from paper_1809_09851_b200 import shard

    dim, n_in, n_out, n_default, desc = CONFIGS[a.config]
    n = a.n or n_default
    prec = 1 if a.prec == "f64" else 0
    esize = 8 if prec else 4
    bytes_per_pt = (n_in + n_out) * esize
    if a.config == "cons2prim1d":
        bytes_per_pt = (n_in + n_out) * esize  # rho read, not written: 3R + 3W
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist = None
    # Under torchrun (WORLD_SIZE set) the process group is initialised even
    # for one rank, so the barrier / max-over-ranks / allreduce code is the
    # same at N = 1 as at N = 8.
    if world > 1 or "WORLD_SIZE" in os.environ:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    outs = None
    stream = torch.cuda.Stream(device=dev)
    first, _ = shard.weak_slice(rank, n)  # weak scaling: global slice [r*n, (r+1)*n)
    dt = torch.float64 if prec else torch.float32

    with torch.cuda.stream(stream):
        if a.config == "axpy":
            x = fvb.synth_uniform(n, prec=prec, seed=1, first=first)
            y = fvb.synth_uniform(n, prec=prec, seed=1, first=world * n + first)
            ins = [x, y]
            outs = [y]
        elif a.config == "eos":  # rho and rho*E of the random state, as rho and e
            st = fvb.synth_state(1, n, prec=prec, seed=0x5EED, first=first)
            ins = [st[0], st[2]]
            outs = [torch.empty(n, dtype=dt, device=dev) for _ in range(2)]
        else:
            ins = fvb.synth_state(dim, n, prec=prec, seed=0x5EED, first=first)
            outs = [torch.empty(n, dtype=dt, device=dev) for _ in range(n_out)]
        lam = torch.empty((), dtype=dt, device=dev)
        lam_global = torch.empty((), dtype=torch.float64, device=dev)

    def step():
        if a.config == "flux3d":
            fvb.flux(ins, dim, out=outs, stream=stream)
        elif a.config == "cons2prim1d":
            fvb.cons2prim(ins, dim, out=outs, stream=stream)
        elif a.config == "jacobian3d":
            fvb.jacobian(ins, dim, out=outs, lambda_max=lam, stream=stream)
        elif a.config == "vmag2":
            fvb.v_mag2(ins, dim, out=outs[0], stream=stream)
        elif a.config == "prim2cons3d":  # the state's planes read as [rho, v, p]
            fvb.prim2cons(ins, dim, out=outs, stream=stream)
        elif a.config == "flux_prim3d":
            fvb.flux_prim(ins, dim, out=outs, stream=stream)
        elif a.config == "eos":
            fvb.eos(ins[0], ins[1], p=outs[0], T=outs[1], stream=stream)
        elif a.config == "cfl3d":
            fvb.wave_speed_max(ins, dim, lambda_max=lam, stream=stream)
        else:
            fvb.axpy_sin(ins[0], ins[1], stream=stream)

    def allreduce():
        # the path's one real exchange: CFL max over GPUs (NCCL over NVLink)
        if a.config == "jacobian3d" and dist is not None:
            with torch.cuda.stream(stream):
                lam_global.copy_(lam)
                shard.allreduce_max(lam_global)

    for _ in range(a.warmup):
        step()
        allreduce()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()

    k_start = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    k_end = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(torch.cuda.current_device())
    # A working set that fits twice into L2 (C1: 24 MB per step) would be
    # re-read from L2 on every step: flush L2 between timed steps (a 256 MB
    # write, then a read of it so the step does not pay for write-backs of
    # the flush's own dirty lines; outside each step's event pair) and time
    # each step on its own.
    # --l2-warm instead replays the K steps back to back as one CUDA graph
    # (the time-stepping-loop case; labelled as such, never the default).
    ws_bytes = n * bytes_per_pt
    flush_l2 = ws_bytes < 2 * L2_BYTES and not a.l2_warm
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush_l2 else None
    flush_sum = torch.empty((), dtype=torch.int64, device=dev)
    graph = None
    if a.l2_warm:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for _ in range(a.steps):
                step()
        torch.cuda.synchronize()
    with sampler:
        with torch.cuda.stream(stream):
            t0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                for i in range(a.steps):
                    if flush is not None:
                        flush.zero_()       # evicts our planes from L2 ...
                        flush_sum.copy_(flush.view(torch.int64).sum())  # ... and cleans it
                    k_start[i].record(stream)
                    step()
                    k_end[i].record(stream)
                    allreduce()
            t1.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    elapsed_ms = t0.elapsed_time(t1)
    if graph is not None:
        kern_avg = elapsed_ms / a.steps
    else:
        kernel_ms = [s.elapsed_time(e) for s, e in zip(k_start, k_end)]
        kern_avg = sum(kernel_ms) / len(kernel_ms)
        if flush is not None:  # the timed region is the K steps, not the flushes
            elapsed_ms = sum(kernel_ms)
    if flush_l2:
        l2_note = ("working set %.0f MB < 2x L2: L2 flushed (256 MB write + read) between "
                   "timed steps, each step timed by its own events" % (ws_bytes / 1e6))
    elif a.l2_warm:
        l2_note = ("L2-warm: %d steps replayed back to back as one CUDA graph, working set "
                   "%.0f MB (not flushed)" % (a.steps, ws_bytes / 1e6))
    else:
        l2_note = "inputs larger than L2 (%.1f GB per GPU vs 126 MB)" % (n * n_in * esize / 1e9)

    if dist is not None:
        tt = torch.tensor([elapsed_ms, kern_avg], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms, kern_avg = tt.tolist()

    # ---- end to end through the host-buffer C-ABI call -----------------------------
    e2e = None
    if not a.no_e2e and a.config not in ("axpy", "eos", "cfl3d"):
        try:
            e2e = end_to_end(a, fvb, ins, n, n_in, n_out, dim, dt, esize, local, dist, world,
                             dev, torch)
        except (RuntimeError, MemoryError) as ex:  # e.g. pinned host memory exhausted
            e2e = {"value": None, "unit": "Gpoints/s", "unavailable": str(ex)[:200]}

    # ---- CPU baseline (rank 0, N=1 only) --------------------------------------------
    cpu = None
    if not a.no_cpu_baseline and world == 1 and rank == 0:
        try:
            threads = cpu_threads()
            sample = min(n, a.cpu_sample if a.config != "axpy" else n)
            if a.config == "jacobian3d":
                sample = min(sample, 2_000_000)
            # a probe rep sizes the run to about a.cpu_seconds of CPU work
            _, probe = reference_run(a.config, a.prec, 1, 1, sample, threads)
            reps = int(min(500, max(3, a.cpu_seconds / max(probe[0] * 1e-9, 1e-6))))
            pts, times = reference_run(a.config, a.prec, reps, 1, sample, threads)
            med = statistics.median(times)
            cpu = {"value": pts / (med * 1e-9) / 1e9, "unit": "Gpoints/s", "cores": threads,
                   "kind": "reference",
                   "sample": f"{pts} points of the same workload per rep, median of {reps} reps "
                             f"({sum(times) * 1e-9:.1f} s of CPU work) after 1 JIT warm-up, "
                             f"Backend::parallel(0, {threads})"}
        except Exception as ex:  # reported, never a substitute for the device number
            cpu = {"value": None, "unit": "Gpoints/s", "cores": cpu_threads(),
                   "kind": "reference", "sample": f"unavailable: {ex}"}

    peak, peak_src = measured_peak()
    achieved = bytes_per_pt * n / (kern_avg * 1e-3) / 1e9
    ms_per_step = elapsed_ms / a.steps
    value = world * n / (ms_per_step * 1e-3) / 1e9
    clocks = sampler.summary()
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "Gpoints/s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": a.prec,
        "data": "synthetic (on-device SplitMix64 random_state of acceptance.cpp:214-230, "
                "seed 0x5eed, bit-identical to the reference generator)",
        "config": {"workload": desc, "config": a.config, "points_per_gpu": n,
                   "global_points": world * n, "dim": dim, "precision": a.prec,
                   "bytes_per_point": bytes_per_pt,
                   "l2": l2_note,
                   "parallelism": f"index-range shards x{world}" + (
                       " + NCCL allreduce-max" if a.config == "jacobian3d" and world > 1 else "")},
        "hbm_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_src,
                     "frac_of_nominal_8000": achieved / 8000.0,
                     "traffic": profiled_traffic(a.config, a.prec, n),
                     "kernel_ms": kern_avg},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": a.steps,
        "clocks": clocks,
    }
    if dist is not None:
        dist.destroy_process_group()
    return line


def main():
    a = parse()
    rank, world, local = dist_env()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched directly with --gpus N: re-launch as N ranks, one per GPU,
        # exactly as the driver does
        import socket
        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        # (--n is spelled --points: torchrun's parser would take "--n" as an
        # ambiguous prefix of its own options)
        args = ["--points" + x[3:] if x == "--n" or x.startswith("--n=") else x
                for x in sys.argv[1:]]
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
                                  "--master-port", str(port), os.path.abspath(__file__)] + args)
    if "WORLD_SIZE" in os.environ and a.gpus != world:
        print(f"bench: --gpus {a.gpus} but WORLD_SIZE={world}; using {world}", file=sys.stderr)
    # stdout carries exactly one JSON line: everything else any library
    # prints to fd 1 (e.g. NCCL's version banner at init) goes to stderr.
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    if a.impl == "reference":
        if rank != 0:
            return 0
        dim, n_in, n_out, n_default, desc = CONFIGS[a.config]
        threads = cpu_threads()
        sample = min(a.n or n_default, a.cpu_sample)
        if a.config == "jacobian3d":
            sample = min(sample, 2_000_000)
        # bounded: shrink the per-step sample if the run would exceed ~3 minutes
        pts, t_probe = reference_run(a.config, a.prec, 1, 1, sample, threads)
        est = t_probe[0] * 1e-9 * (a.steps + a.warmup)
        if est > 180:
            sample = max(100_000, int(sample * 180 / est))
        pts, times = reference_run(a.config, a.prec, a.steps, a.warmup, sample, threads)
        ms = statistics.mean(times) * 1e-6
        value = pts / (ms * 1e-3) / 1e9
        esize = 8 if a.prec == "f64" else 4
        line = {
            "metric": METRIC, "value": value, "unit": "Gpoints/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": a.prec,
            "data": "synthetic (random_state of acceptance.cpp:214-230, seed 0x5eed)",
            "config": {"workload": desc, "config": a.config, "points_per_step": pts,
                       "bytes_per_point": (n_in + n_out) * esize,
                       "parallelism": f"reference Backend::parallel(0, {threads}) on host cores"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "Gpoints/s", "cores": threads,
                             "kind": "reference",
                             "sample": f"{pts} points per step (bounded sample of the "
                                       f"{a.n or n_default}-point workload), unmodified "
                                       f"reference evaluate_block/evaluate with its runtime JIT"},
            "e2e": {"value": value, "unit": "Gpoints/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
    else:
        line = device_run(a, rank, world, local)
    if rank == 0:
        text = json.dumps(line)
        sys.stdout.flush()
        os.write(json_fd, (text + "\n").encode())
        if a.out:
            with open(a.out, "a") as f:
                f.write(text + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
