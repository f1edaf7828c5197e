#!/usr/bin/env python3
"""The same block expression through its hand-written fused kernel and through
the general NVRTC lowering (fvb_lookup with FVB_FORCE_LOWER=1), on one B200.

    python tools/lowered_vs_handwritten.py [--n 100000000]

Prints one JSON line per block: the key's kernel name, time per launch and
HBM GB/s for both paths, and whether their outputs are bitwise equal.
The lowered run happens in a child process, because FVB_FORCE_LOWER is read
once per process.
"""

import argparse
import json
import os
import re
import struct
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONSTS = {"half": 0.5, "gm1": 0.4, "gamma": 1.4, "cv": 2.5, "zero": 0.0, "one": 1.0}
BLOCKS = {"flux3_f64": (3, 5, 15), "jacobian3_f64": (3, 5, 75), "cons2prim_c1_f64": (1, 3, 3)}


def key_of(pattern):
    def sub(m):
        v = CONSTS[m.group(2)]
        return "C%s%016x;" % (m.group(1), struct.unpack("<Q", struct.pack("<d", v))[0])
    return re.sub(r"C([sd])#(\w+);", sub, pattern)


def run_one(name, n, dump, slot_map):
    import ctypes

    import numpy as np
    import torch

    import paper_1809_09851_b200 as fvb
    from paper_1809_09851_b200 import _native as N

    dim, nin, nout = BLOCKS[name]
    k = fvb.lookup(key_of(dict(fvb.patterns())[name]))
    state = fvb.synth_state(dim, n, seed=0x5EED)
    outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(nout)]
    # canonical plane c -> argument slot, from the hand-written kernel's
    # in_slot (the key's first-appearance leaf order; a lowered kernel takes
    # its arguments in that same slot order)
    slots = [None] * k.n_inputs
    for c in range(nin):
        slots[slot_map[c]] = state[c]
    args = N.ptr_array([t.data_ptr() for t in outs + slots])
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        N.check(k.fn(ctypes.byref(k), 0, n, args, s))
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    reps = 20
    ev[0].record()
    for _ in range(reps):
        N.check(k.fn(ctypes.byref(k), 0, n, args, s))
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    if dump:
        np.save(dump, np.stack([t[:: max(1, n // 65536)].cpu().numpy() for t in outs]))
    return {"kernel": k.name.decode(), "ms": ms,
            "GBps": (nin + nout) * 8 * n / (ms * 1e-3) / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--child", default="")
    ap.add_argument("--dump", default="")
    ap.add_argument("--slots", default="")
    a = ap.parse_args()
    if a.child:
        print(json.dumps(run_one(a.child, a.n, a.dump, [int(x) for x in a.slots.split(",")])))
        return
    import numpy as np

    import paper_1809_09851_b200 as fvb

    for name in BLOCKS:
        n = a.n if name != "jacobian3_f64" else a.n // 4
        res = {}
        hw = fvb.lookup(key_of(dict(fvb.patterns())[name]))
        slot_map = ",".join(str(hw.in_slot[c]) for c in range(BLOCKS[name][1]))
        for mode, env in (("handwritten", {}), ("lowered", {"FVB_FORCE_LOWER": "1"})):
            dump = f"/tmp/lvh_{name}_{mode}.npy"
            p = subprocess.run([sys.executable, __file__, "--child", name, "--n", str(n),
                                "--dump", dump, "--slots", slot_map], capture_output=True, text=True,
                               env={**os.environ, **env})
            if p.returncode != 0:
                res[mode] = {"error": p.stderr[-400:]}
                continue
            res[mode] = json.loads(p.stdout.strip().splitlines()[-1])
        try:
            a0 = np.load(f"/tmp/lvh_{name}_handwritten.npy")
            a1 = np.load(f"/tmp/lvh_{name}_lowered.npy")
            res["bitwise_equal_sampled"] = bool(a0.tobytes() == a1.tobytes())
        except Exception as ex:  # noqa: BLE001
            res["bitwise_equal_sampled"] = f"n/a: {ex}"
        print(json.dumps({"block": name, "n": n, **res}), flush=True)


if __name__ == "__main__":
    main()
