"""The N>1 host logic on CPU: contiguous slices tile the range exactly for
ragged N, and the CFL maximum reduced across 2 gloo ranks equals the global
maximum bit for bit (the path's one collective; NCCL on the B200 box)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1809_09851_b200 import shard


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [0, 1, 2, 7, 1000, 10**8 + 3])
def test_slices_tile_the_range(world, n):
    prev_hi = 0
    for r in range(world):
        lo, hi = shard.slice_bounds(r, world, n)
        assert lo == prev_hi and hi >= lo
        assert hi - lo in (n // world, n // world + 1)
        prev_hi = hi
    assert prev_hi == n


def test_slice_bounds_rejects_bad_rank():
    with pytest.raises(ValueError):
        shard.slice_bounds(2, 2, 10)


def test_weak_slices_are_disjoint_and_contiguous():
    n = 1000
    spans = [shard.weak_slice(r, n) for r in range(8)]
    assert spans[0] == (0, n) and all(spans[i][1] == spans[i + 1][0] for i in range(7))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_total, dim, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle

    orc = oracle.oracle()
    lo, hi = shard.slice_bounds(rank, world, n_total)
    # each rank generates its own slice from the global index, exactly as the
    # device generator does on each GPU
    s = orc.random_state(dim, hi - lo, seed=0x5EED, first=lo)
    local = orc.wave_speed_max(dim, s) if hi > lo else 0.0
    t = torch.tensor([local], dtype=torch.float64)
    shard.allreduce_max(t)
    result[rank] = t.item()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_total", [(2, 1), (2, 10_001), (3, 10_001), (8, 10_001),
                                           (8, 5)])
def test_cfl_allreduce_max_gloo(orc, world, n_total):
    # ragged slices (N mod G != 0, and N < G: empty ranks) reduce to the
    # single-process maximum bit for bit on every rank
    dim = 3
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n_total, dim, result), nprocs=world, join=True)
    whole = orc.wave_speed_max(dim, orc.random_state(dim, n_total, seed=0x5EED))
    assert [result[r] for r in range(world)] == [whole] * world
    # and bitwise: the global max is one of the per-point values
    assert np.float64(whole).tobytes() == np.float64(result[0]).tobytes()


def _nan_worker(rank, world, port, values, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for case in values:
        for dt in (torch.float64, torch.float32):
            t = torch.tensor([case[rank]], dtype=dt)
            shard.allreduce_max(t)
            out.append(t.view(torch.int64 if dt == torch.float64 else torch.int32).item())
    result[rank] = out
    dist.destroy_process_group()


def test_cfl_allreduce_is_the_unsigned_bit_max(orc):
    # the cross-rank max follows the device reduction: IEEE bits compared as
    # unsigned integers, so a NaN on any rank reaches every rank, inf beats
    # every finite speed, and +0 < every positive speed
    nan, inf = float("nan"), float("inf")
    cases = [(1.5, 2.5), (2.5, 1.5), (nan, 3.0), (3.0, nan), (inf, 7.0), (0.0, 1e-300),
             (0.0, 0.0), (-nan, 1.0)]
    world = 2
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_nan_worker, args=(world, _free_port(), cases, result), nprocs=world, join=True)
    want = []
    for case in cases:
        for np_t, ui in ((np.float64, np.uint64), (np.float32, np.uint32)):
            bits = [int(np.array([v], np_t).view(ui)[0]) for v in case]
            b = max(bits)
            want.append(int(np.array([b], ui).view(np.int64 if ui == np.uint64 else np.int32)[0]))
    assert result[0] == result[1] == want
