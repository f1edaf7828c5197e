#!/usr/bin/env python3
"""CSR block matvec on one B200 against its roofline and the
reference's serial csr_matvec_acc.

    python tools/csr_bench.py [--n 256] [--reps 20]

Workload: the 7-point Laplacian on an n^3 grid (y += A x, f64), the PDE
stencil the block layer's matvec serves.  Algorithmic bytes per launch:
row_ptr 8*(rows+1) + (values + col_idx) 16*nnz + x 8*rows (each element
once) + y 16*rows (read + write).  Prints one JSON line per kernel variant
(FVB_CSR_MODE=row|warp forces one form; unset = the library's
own choice) and the reference's rate on a bounded sample.
Parity: the device y equals the oracle bit for bit.
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ref-n", type=int, default=96)
    a = ap.parse_args()
    import torch

    import oracle
    import paper_1809_09851_b200 as fvb
    from paper_1809_09851_b200 import _native as N
    from tests.test_parity_gpu import stencil7

    dev = torch.device("cuda", 0)
    rp, ci, v = stencil7(a.n)
    rows, nnz = len(rp) - 1, len(ci)
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, rows)
    y0 = np.zeros(rows)
    drp = torch.from_numpy(rp.view(np.int64)).to(dev)
    dci64 = torch.from_numpy(ci.view(np.int64)).to(dev)
    dv = torch.from_numpy(v).to(dev)
    dx = torch.from_numpy(x).to(dev)
    dy = torch.zeros(rows, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    want = oracle.oracle().csr_matvec_acc(rp, ci, v, x, y0)
    peak = 6548.2
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    variant = os.environ.get("FVB_CSR_MODE", "") or (
        "rowwise" if os.environ.get("FVB_CSR_ROWWISE", "0") not in ("", "0") else "auto")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > L2 between reps
    # the reference's 64-bit size_t indices, then the 32-bit device layout
    # DeviceCsr keeps (fvb_csr_matvec_acc_u32): 16 vs 12 bytes per nonzero
    for width, dci, fn in ((8, dci64, N.lib().fvb_csr_matvec_acc),
                           (4, dci64.to(torch.int32), N.lib().fvb_csr_matvec_acc_u32)):
        def launch():
            N.check(fn(1, 1, rows, nnz, drp.data_ptr(), dci.data_ptr(), dv.data_ptr(),
                       dx.data_ptr(), dy.data_ptr(), stream.cuda_stream))

        dy.zero_()
        launch()
        torch.cuda.synchronize()
        bitwise = dy.cpu().numpy().tobytes() == want.tobytes()
        for _ in range(3):
            launch()
        times = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            launch()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e-3)
        t = float(np.median(times))
        bytes_ = 8 * (rows + 1) + (8 + width) * nnz + 8 * rows + 16 * rows
        line = {"kernel": f"csr_{variant}" + ("" if width == 8 else "_u32"), "grid": f"{a.n}^3",
                "rows": rows, "nnz": nnz, "index_bytes": width,
                "ms": t * 1e3, "grows_per_s": rows / t / 1e9, "algorithmic_bytes": bytes_,
                "GBps": bytes_ / t / 1e9, "peak_GBps": peak, "frac": bytes_ / t / 1e9 / peak,
                "bitwise_vs_oracle": bitwise, "l2": "flushed between reps"}
        print(json.dumps(line), flush=True)
    ref = oracle.reference()
    if ref is not None and variant == "auto" and a.ref_n > 0:
        ts, rnnz = ref.time_csr(a.ref_n, 5)
        rrows = a.ref_n ** 3
        print(json.dumps({"kernel": "reference csr_matvec_acc (serial, 1 core)",
                          "grid": f"{a.ref_n}^3", "rows": rrows, "nnz": rnnz,
                          "ms": float(np.median(ts)) * 1e3,
                          "grows_per_s": rrows / float(np.median(ts)) / 1e9}), flush=True)
    del fvb


if __name__ == "__main__":
    main()
