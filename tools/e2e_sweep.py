#!/usr/bin/env python3
"""The end-to-end (host-buffer) path against its own ceiling: PCIe.

    python tools/e2e_sweep.py [--n 100000000]

1. Measures the link: pinned host<->device copy bandwidth, each direction
   alone and both at once (cudaMemcpyAsync on two streams).
2. Times fvb_flux_host (3-D flux, fp64) for several pipeline chunk sizes.
3. Prints the e2e roofline: the flux moves 40 B/pt H2D and 96 B/pt D2H
   (row 0 is copied host-side); the two directions overlap, so the
   ceiling is the D2H side: 96 B/pt at the bidirectional D2H rate.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000_000)
    a = ap.parse_args()
    import torch

    import paper_1809_09851_b200 as fvb

    n = a.n
    gb = 2 << 30
    h = torch.empty(gb // 8, dtype=torch.float64).pin_memory()
    h2 = torch.empty(gb // 8, dtype=torch.float64).pin_memory()
    d = torch.empty(gb // 8, dtype=torch.float64, device="cuda")
    d2 = torch.empty(gb // 8, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / reps

    h2d = gb / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9
    d2h = gb / timed(lambda: h.copy_(d, non_blocking=True)) / 1e9

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    both_s = timed(both)
    link = {"h2d_GBps": h2d, "d2h_GBps": d2h, "bidir_each_GBps": gb / both_s / 1e9}
    print(json.dumps({"link": link}), flush=True)
    del h, h2, d, d2

    state = fvb.synth_state(3, n, seed=0x5EED)
    hin = torch.empty((5, n), dtype=torch.float64).pin_memory()
    for i, t in enumerate(state):
        hin[i].copy_(t)
    hin = list(hin.unbind(0))
    hout = list(torch.empty((15, n), dtype=torch.float64).pin_memory().unbind(0))
    del state
    torch.cuda.empty_cache()
    bidir = link["bidir_each_GBps"]
    ceil_gpts = 1.0 / (96 / (bidir * 1e9)) / 1e9
    # pageable host planes: the bounce buffers and copy threads
    pin_in = [t.clone() for t in hin]
    pin_out = [t.clone() for t in hout]
    ctx = fvb.HostContext(0)
    s = timed(lambda: ctx.flux(pin_in, 3, pin_out), reps=3)
    ctx.close()
    print(json.dumps({"chunk_points": "default, PAGEABLE host planes", "ms": s * 1e3,
                      "gpts": n / s / 1e9}), flush=True)
    del pin_in, pin_out
    for chunk in (1 << 20, 1 << 22, 1 << 24, 0):
        ctx = fvb.HostContext(0, chunk_points=chunk)
        s = timed(lambda: ctx.flux(hin, 3, hout), reps=3)
        ctx.close()
        print(json.dumps({"chunk_points": chunk or "default(256 MiB/slot)", "ms": s * 1e3,
                          "gpts": n / s / 1e9, "ceiling_gpts_at_bidir_link": ceil_gpts,
                          "frac_of_ceiling": n / s / 1e9 / ceil_gpts}), flush=True)


if __name__ == "__main__":
    main()
