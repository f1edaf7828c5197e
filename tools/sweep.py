#!/usr/bin/env python3
"""C5: size sweep of the fused 3-D flux kernel on one B200, N = 1e3 ... 1e9,
beside the unmodified reference on the host cores, with CSV records in the
reference's own schema (proj/src/bench.cpp:423-443).

    python tools/sweep.py [--prec f64] [--max 1e9] [--out gpurun_out/sweep_c5]

Writes <out>.jsonl (one record per size) and <out>.csv:

* a `b200x1` row per size: the device median time (CUDA events, after
  warm-up);
* a `parallel` row: the reference on all host threads, up to --ref-max points;
* the reference's own `run_miniapp` record at N = 2^24 (its published-by-
  harness figure).

The mflops and bandwidth_mbs columns use the reference's tree-derived
accounting: one flop per op node, reads = distinct leaves per item, plus one
write per item.  That is 528 B/pt for the 3-D flux, against the fused kernel's
160 algorithmic B/pt, which the JSON records separately.  For device rows,
overhead_ratio = device time / HBM-roofline time at the measured copy peak.
For the reference's own record it is its generic/hand-fused ratio.  N = 2e9
fp64 needs 320 GB and so >= 2 GPUs; it is listed as infeasible at G = 1 (f32, 160 GB, runs).
"""

import argparse
import json
import os
import re
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def tree_accounting(pattern: str, width: int):
    """(flops/pt, bytes/pt) of the reference's miniapp accounting from a
    registry pattern (bench.cpp:347-357)."""
    body = pattern.split(":", 1)[1]
    flops = 0
    nbytes = 0
    for item in body.split("|"):
        flops += len(re.findall(r"[UB]\d+[sd]\(", item))
        leaves = set(re.findall(r"L[sd](\d+);", item))
        nbytes += (len(leaves) + 1) * width
    return flops, nbytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prec", default="f64", choices=["f64", "f32"])
    ap.add_argument("--max", type=float, default=1e9)
    ap.add_argument("--ref-max", type=float, default=1e7)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep_c5"))
    a = ap.parse_args()

    import torch

    import oracle
    import paper_1809_09851_b200 as fvb
    from bench import measured_peak

    prec = 1 if a.prec == "f64" else 0
    w = 8 if prec else 4
    dt = torch.float64 if prec else torch.float32
    pattern = dict(fvb.patterns())[f"flux3_{a.prec}"]
    tflops, tbytes = tree_accounting(pattern, w)
    alg_bytes = 20 * w
    peak, _ = measured_peak()
    R = oracle.reference()
    threads = len(os.sched_getaffinity(0))
    sizes = [int(10 ** e) for e in range(3, 10) if 10 ** e <= a.max]
    # 5e8, and 2e9 where its 20 planes fit this GPU (f32: 160 GB of 180;
    # f64 needs 320 GB, i.e. >= 2 GPUs)
    free = torch.cuda.mem_get_info()[0]
    for extra in (int(5e8), int(2e9)):
        if extra <= a.max and (extra < int(2e9) or 20 * w * extra < free - (2 << 30)):
            sizes.append(extra)
    sizes = sorted(set(sizes))
    recs, csv = [], []
    stream = torch.cuda.Stream()
    for n in sizes:
        rec = {"n": n, "prec": a.prec, "gpus": 1}
        try:
            with torch.cuda.stream(stream):
                s = fvb.synth_state(3, n, prec=prec, seed=0x5EED)
                out = [torch.empty(n, dtype=dt, device="cuda") for _ in range(15)]
            reps = int(min(2000, max(20, 2e9 / max(n, 1) / 10)))
            for _ in range(5):
                fvb.flux(s, 3, out=out, stream=stream)
            torch.cuda.synchronize()
            if n <= 1_000_000:
                # Launch-bound sizes: time a CUDA graph of 100 back-to-back
                # launches (what a native caller issuing a time loop sees),
                # not the Python-ctypes gap between launches.
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for _ in range(100):
                        fvb.flux(s, 3, out=out, stream=stream)
                ts = []
                for _ in range(max(5, reps // 100)):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(
                        enable_timing=True)
                    with torch.cuda.stream(stream):  # replay() runs on the current stream
                        e0.record(stream)
                        g.replay()
                        e1.record(stream)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e-3 / 100)
                ts.sort()
                rec["timing"] = "CUDA graph of 100 launches"
                del g
            else:
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(reps)]
                for e0, e1 in ev:
                    e0.record(stream)
                    fvb.flux(s, 3, out=out, stream=stream)
                    e1.record(stream)
                torch.cuda.synchronize()
                ts = sorted(e0.elapsed_time(e1) * 1e-3 for e0, e1 in ev)
                rec["timing"] = "CUDA events per launch"
            med = statistics.median(ts)
            rec.update({"reps": reps, "median_s": med, "best_s": ts[0],
                        "gpts": n / med / 1e9, "GBps": alg_bytes * n / med / 1e9,
                        "frac_of_measured": alg_bytes * n / med / 1e9 / peak,
                        "roofline_s": alg_bytes * n / (peak * 1e9)})
            csv.append(f"miniapp,b200x1,{a.prec},{n},{med * 1e9:.3f},"
                       f"{tflops * n / med / 1e6:.3f},{tbytes * n / med / 1e6:.3f},"
                       f"{med / rec['roofline_s']:.4f}")
            del s, out
            torch.cuda.empty_cache()
        except torch.cuda.OutOfMemoryError as ex:
            rec["infeasible"] = f"out of device memory: {str(ex)[:80]}"
            torch.cuda.empty_cache()
        if R is not None and n <= a.ref_max:
            reps = 3 if n >= 1e6 else 10
            t = R.time_config(0, 3, a.prec, n, threads, reps + 1)[1:]
            med_c = statistics.median(t) * 1e-9
            rec.update({"ref_median_s": med_c, "ref_gpts": n / med_c / 1e9, "ref_threads": threads,
                        "speedup": med_c / rec["median_s"] if "median_s" in rec else None})
            csv.append(f"miniapp,parallel,{a.prec},{n},{med_c * 1e9:.3f},"
                       f"{tflops * n / med_c / 1e6:.3f},{tbytes * n / med_c / 1e6:.3f},nan")
        recs.append(rec)
        print(json.dumps(rec), flush=True)
    if int(2e9) not in sizes:
        recs.append({"n": 2_000_000_000, "prec": a.prec, "gpus": 1,
                     "infeasible": f"needs {20 * w * 2} GB of planes ({a.prec}): more than one "
                                   f"GPU's {free / 1e9:.0f} GB free"})
    if R is not None:
        med_ns, ratio = R.run_miniapp(a.prec, 1 << 24, threads)
        csv.append(f"miniapp,parallel,{a.prec},{1 << 24},{med_ns:.3f},"
                   f"{tflops * (1 << 24) / med_ns * 1e3:.3f},"
                   f"{tbytes * (1 << 24) / med_ns * 1e3:.3f},{ratio:.4f}")
        recs.append({"reference_run_miniapp": {"n": 1 << 24, "median_ns": med_ns,
                                               "overhead_ratio": ratio, "threads": threads}})
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out + ".jsonl", "w") as f:
        for r in recs:
            f.write(json.dumps(r) + "\n")
    with open(a.out + ".csv", "w") as f:
        f.write(f"# miniapp accounting: tree-derived; one flop per op node, reads = distinct "
                f"leaves per item, plus one write per item ({tflops} flops, {tbytes} B per "
                f"point)\n")
        f.write("# b200x1 rows: fused sm_100a kernel, CUDA-event median; overhead_ratio = "
                "time / HBM-roofline time at the measured copy peak\n")
        f.write("suite,backend,precision,n,median_ns,mflops,bandwidth_mbs,overhead_ratio\n")
        for line in csv:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
