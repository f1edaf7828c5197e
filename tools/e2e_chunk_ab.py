#!/usr/bin/env python3
"""A/B of the host-buffer pipeline's chunk size on one box: fvb_flux_host
(3-D flux f64, N = 1e8, pinned), chunk sizes interleaved over several rounds
so box drift hits every variant alike.  One JSON line per measurement."""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1809_09851_b200 as fvb

    n = 100_000_000
    s = fvb.synth_state(3, n)
    hin = list(torch.empty((5, n), dtype=torch.float64).pin_memory().unbind(0))
    for a, b in zip(hin, s):
        a.copy_(b)
    hout = list(torch.empty((15, n), dtype=torch.float64).pin_memory().unbind(0))
    del s
    torch.cuda.empty_cache()
    chunks = [0, 2_097_152, 4_194_304, 8_388_608]
    ctxs = {c: fvb.HostContext(0, chunk_points=c) for c in chunks}
    for c in chunks:
        ctxs[c].flux(hin, 3, hout)  # staging allocation
    for rnd in range(4):
        for c in chunks:
            t = time.perf_counter()
            for _ in range(2):
                ctxs[c].flux(hin, 3, hout)
            ms = (time.perf_counter() - t) / 2 * 1e3
            print(json.dumps({"round": rnd, "chunk_points": c or "default(256 MiB/slot)",
                              "ms": ms, "gpts": n / ms / 1e6}), flush=True)


if __name__ == "__main__":
    main()
