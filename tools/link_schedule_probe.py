#!/usr/bin/env python3
"""The e2e flux's PCIe floor, independent of the pipeline: the same bytes as
fvb_flux_host moves at N = 1e8 f64 (4 GB host->device, 9.6 GB device->host,
in 13.4 MB pieces, pinned), on the copy engines alone:
  1. device->host alone, 2. host->device alone,
  3. both directions at once (two streams, everything enqueued),
  4. the same with the host->device pieces issued first on their stream.
If 3 is well below the pipeline's time, the pipeline leaves link time unused."""

import json
import time


def main():
    import torch

    piece = 1_677_721 * 8  # one plane of one default chunk
    up_n, down_n = 300, 720  # 4.0 GB and 9.7 GB
    pool = 64
    h_up = [torch.empty(piece // 8, dtype=torch.float64).pin_memory() for _ in range(pool)]
    h_dn = [torch.empty(piece // 8, dtype=torch.float64).pin_memory() for _ in range(pool)]
    d_up = [torch.empty(piece // 8, dtype=torch.float64, device="cuda") for _ in range(pool)]
    d_dn = [torch.empty(piece // 8, dtype=torch.float64, device="cuda") for _ in range(pool)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def up():
        with torch.cuda.stream(s1):
            for i in range(up_n):
                d_up[i % pool].copy_(h_up[i % pool], non_blocking=True)

    def down():
        with torch.cuda.stream(s2):
            for i in range(down_n):
                h_dn[i % pool].copy_(d_dn[i % pool], non_blocking=True)

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        return best * 1e3

    res = {"piece_MB": piece / 1e6, "up_GB": up_n * piece / 1e9, "down_GB": down_n * piece / 1e9}
    res["down_alone_ms"] = timed(down)
    res["up_alone_ms"] = timed(up)

    def both():
        up()
        down()

    res["both_ms"] = timed(both)

    def interleaved():  # one up piece per 2.4 down pieces, on two streams, as the pipeline does
        with torch.cuda.stream(s1):
            pass
        j = 0
        for i in range(down_n):
            if j < up_n and j * down_n <= i * up_n:
                with torch.cuda.stream(s1):
                    d_up[j % pool].copy_(h_up[j % pool], non_blocking=True)
                j += 1
            with torch.cuda.stream(s2):
                h_dn[i % pool].copy_(d_dn[i % pool], non_blocking=True)

    res["interleaved_ms"] = timed(interleaved)
    res["flux_gpts_at_both"] = 1e8 / res["both_ms"] / 1e6
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
