#!/usr/bin/env python3
"""The reference's CPU path on this host, both backends BASELINE.md §2 names:
Backend::scalar_ref() on one core and Backend::parallel(0, nproc), JIT on,
for every config (bounded samples), plus the serial CSR matvec.

    python tools/ref_cpu.py > profiles/r01_reference_cpu.jsonl

One JSON line per (config, backend): points per rep, median seconds,
Gpoints/s.  Reps follow the reference's decide_reps spirit: one JIT warm-up,
then at least 3 reps.
"""

import json
import os
import platform
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (the reference build, test/bench infrastructure)

# (config, which, dim, prec, sample points for scalar_ref, for parallel)
CASES = [
    ("axpy", 3, 1, "f64", 1_000_000, 1_000_000),
    ("cons2prim1d", 1, 1, "f64", 4_000_000, 20_000_000),
    ("flux3d", 0, 3, "f64", 2_000_000, 10_000_000),
    ("flux3d", 0, 3, "f32", 2_000_000, 10_000_000),
    ("jacobian3d", 2, 3, "f64", 500_000, 2_000_000),
    ("jacobian3d", 2, 3, "f32", 500_000, 2_000_000),
    ("vmag2", 4, 3, "f64", 4_000_000, 20_000_000),
]


def main():
    R = oracle.reference()
    if R is None:
        print(json.dumps({"unavailable": "oracle/_ref/libfvref.so missing"}))
        return 1
    nproc = len(os.sched_getaffinity(0))
    host = {"cpu": platform.processor() or platform.machine(), "nproc": nproc}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                host["cpu"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    print(json.dumps({"host": host}), flush=True)
    for cfg, which, dim, prec, n1, nn in CASES:
        for backend, workers, n in (("scalar_ref", 0, n1), (f"parallel(0,{nproc})", nproc, nn)):
            times = R.time_config(which, dim, prec, n, workers, 4)[1:]
            med = statistics.median(times) * 1e-9
            print(json.dumps({"config": cfg, "prec": prec, "backend": backend, "cores":
                              1 if workers == 0 else nproc, "points": n, "median_s": med,
                              "gpoints_per_s": n / med / 1e9}), flush=True)
    ts, nnz = R.time_csr(96, 4)
    med = statistics.median(ts[1:])
    print(json.dumps({"config": "csr7 96^3", "prec": "f64", "backend": "csr_matvec_acc (serial)",
                      "cores": 1, "points": 96 ** 3, "nnz": nnz, "median_s": med,
                      "gpoints_per_s": 96 ** 3 / med / 1e9}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
