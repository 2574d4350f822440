"""Multi-rank host logic on CPU (gloo, world size 2).

The device path averages a synced range across ranks as: local pairwise
subtree sum -> all-to-all of slices -> pairwise reduction over ranks -> /K ->
all-gather (lab.cu sync_range, DSX_SYNC_PAIRWISE).  This test runs that exact
schedule with two gloo processes on the C oracle's pairwise sums and checks
it is bit-identical to the reference's in-process K-worker mean
(trainer.cpp:31-38, 226-234); it also checks the plan the C-ABI reports and
that the NCCL unique id used to bootstrap the device communicator can be
broadcast from rank 0.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def pairwise(rows):
    """trainer.cpp:31-38 over a list of equal-length arrays."""
    n = len(rows)
    if n == 1:
        return rows[0].copy()
    if n == 2:
        return rows[0] + rows[1]
    mid = n // 2
    return pairwise(rows[:mid]) + pairwise(rows[mid:])


def _worker(rank, world, port, K, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1234)
    W = rng.normal(size=(K, n))  # every rank draws the same global data
    kl = K // world
    mine = W[rank * kl:(rank + 1) * kl]
    part = pairwise(list(mine))                       # local subtree sum
    base, extra = divmod(n, world)
    lo = [r * base + min(r, extra) for r in range(world)]
    cnt = [base + (1 if r < extra else 0) for r in range(world)]
    # all-to-all of slices (gloo all_gather of the whole partial, then pick)
    gathered = [torch.zeros(n, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(part))
    recv = [g.numpy()[lo[rank]:lo[rank] + cnt[rank]] for g in gathered]
    reduced = pairwise(recv) / K                      # rank-ordered pairwise, /K
    slices = [torch.zeros(n, dtype=torch.float64) for _ in range(world)]
    full = np.zeros(n)
    full[lo[rank]:lo[rank] + cnt[rank]] = reduced
    dist.all_gather(slices, torch.from_numpy(full))
    mean = np.zeros(n)
    for r in range(world):
        mean[lo[r]:lo[r] + cnt[r]] = slices[r].numpy()[lo[r]:lo[r] + cnt[r]]
    ref = pairwise(list(W)) / K                       # in-process reference
    ok = bool(np.array_equal(mean, ref))
    # NCCL bootstrap id broadcast (bytes object through gloo)
    from paper_2502_11058_b200.lab import nccl_unique_id
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ok = ok and isinstance(obj[0], bytes) and len(obj[0]) == 128
    out[rank] = int(ok)
    dist.destroy_process_group()


@pytest.mark.parametrize("K,n", [(8, 1001), (2, 17), (4, 4096)])
def test_two_rank_pairwise_sync_is_bit_exact(K, n):
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0, 0])
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, K, n, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert list(out) == [1, 1]


@pytest.mark.parametrize("K,world,exact", [(8, 1, 1), (8, 2, 1), (8, 4, 1), (8, 8, 1),
                                           (6, 2, 1), (6, 3, 0), (12, 4, 1), (12, 3, 0), (16, 4, 1),
                                           (5, 2, 0)])
def test_sync_plan_reports_pairwise_exactness(K, world, exact):
    from paper_2502_11058_b200 import native
    flag = C.c_int(-1)
    native.call("dsx_sync_plan", K, world, C.byref(flag))
    assert flag.value == exact
