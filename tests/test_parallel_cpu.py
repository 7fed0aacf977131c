"""Multi-process (gloo, world_size 2, CPU) checks of the multi-GPU plumbing:
row ownership (runs stay rank-local, balance) and the owner-zeroed all-reduce
used for the per-level flag / mask / count exchange."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_01251_b200.parallel import owner_zero_allreduce, row_owner


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        n = 1000
        j = torch.from_numpy(rng.integers(0, 64, n))
        k = torch.from_numpy(rng.integers(0, 64, n))
        truth_flags = torch.from_numpy(rng.integers(0, 64, n).astype(np.uint8))
        truth_masks = torch.from_numpy(rng.integers(-2**62, 2**62, n).astype(np.int64))
        owner = torch.from_numpy(row_owner(j.numpy(), k.numpy(), 64, world))
        mine = owner == rank
        # every rank starts with garbage where it is not the owner
        flags = torch.where(mine, truth_flags, torch.full_like(truth_flags, 255))
        masks = torch.where(mine, truth_masks, torch.full_like(truth_masks, -1))
        owner_zero_allreduce(flags, mine, dist.ReduceOp.MAX)
        owner_zero_allreduce(masks, mine, dist.ReduceOp.SUM)
        q.put((rank, bool(torch.equal(flags, truth_flags)), bool(torch.equal(masks, truth_masks)),
               int(mine.sum())))
    finally:
        dist.destroy_process_group()


def test_owner_zero_allreduce_gloo_ws2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(r[1] and r[2] for r in res), res
    assert sum(r[3] for r in res) == 1000


def test_row_owner_properties():
    # a run (fixed j,k, varying i) has one owner; rows are balanced
    j, k = np.meshgrid(np.arange(64), np.arange(64), indexing="ij")
    for n in (2, 4, 8):
        o = row_owner(j, k, 64, n)
        counts = np.bincount(o.ravel(), minlength=n)
        assert counts.max() - counts.min() <= 1
        # neighbouring rows in y differ in owner (interleaving)
        assert np.all(o[1:, :] != o[:-1, :])
    assert np.all(row_owner(j, k, 64, 1) == 0)


def test_balanced_row_owner_contiguous_and_balanced():
    from paper_2512_01251_b200.parallel import balanced_row_owner
    rng = np.random.default_rng(3)
    counts = rng.integers(0, 40, 4096) * (rng.random(4096) < 0.3)
    for n in (1, 2, 3, 4, 8):
        own = balanced_row_owner(counts, n)
        assert own.min() >= 0 and own.max() <= n - 1
        assert np.all(np.diff(own.astype(int)) >= 0)  # contiguous row ranges
        load = np.bincount(own, weights=counts, minlength=n)
        assert load.max() - load.min() <= 2 * counts.max()  # balanced to within a row or two
    assert balanced_row_owner(np.zeros(10, int), 4).max() == 0
