#!/usr/bin/env python3
"""The host-buffer pipeline against the link floor (tools/link_schedule_probe.py):
fvb_flux_host (3-D flux f64, N = 1e8, pinned) timed in this process's
configuration (FVB_HOST_SLOTS etc. from the environment), and the same kernel
through fvb_launch_host with the 3 row-0 outputs discarded (marked 2: the
pipeline without the host-side pass-through copies), alternating."""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import ctypes

    import torch

    import paper_1809_09851_b200 as fvb
    from paper_1809_09851_b200 import _native as N
    from bench import registry_key

    n = 100_000_000
    s = fvb.synth_state(3, n)
    hin = list(torch.empty((5, n), dtype=torch.float64).pin_memory().unbind(0))
    for a, b in zip(hin, s):
        a.copy_(b)
    hout = list(torch.empty((15, n), dtype=torch.float64).pin_memory().unbind(0))
    del s
    torch.cuda.empty_cache()
    ctx = fvb.HostContext(0)
    k = fvb.lookup(registry_key(fvb, "flux3_f64"))
    slots = [None] * 5
    for i in range(5):
        slots[k.in_slot[i]] = hin[i]
    planes = hout + slots
    count = len(planes)
    ptrs = N.ptr_array([t.data_ptr() for t in planes])
    prec = (ctypes.c_uint8 * count)(*([1] * count))
    where = (ctypes.c_uint8 * count)(*([2, 2, 2] + [0] * (count - 3)))

    def flux_host():
        ctx.flux(hin, 3, hout)

    def no_passthrough():
        N.check(N.lib().fvb_launch_host(ctx._h, ctypes.byref(k), n, ptrs, prec, where, None, None))

    for f in (flux_host, no_passthrough):
        f()
    res = {"slots": os.environ.get("FVB_HOST_SLOTS", "3")}
    for name, f in (("flux_host_ms", flux_host), ("no_passthrough_ms", no_passthrough)):
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            f()
            best = min(best, time.perf_counter() - t)
        res[name] = best * 1e3
    res["flux_host_gpts"] = n / res["flux_host_ms"] / 1e6
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
