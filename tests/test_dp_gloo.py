"""Host-side logic of the multi-GPU path on CPU: world_size 2 over gloo.

The device kernels need a B200; what runs here is the data-parallel plumbing
they rely on: the all-reduce of int64 cross terms wraps mod 2^64 exactly like
the ring, shard rows partition the batch, and shard offsets place each
rank's PRF words at its contiguous range of the reference's flat tensor."""

import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_10949_b200.engine import TrioSession
from paper_2104_10949_b200.nn import DataParallel


def _port():
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
        dp = DataParallel.from_process_group()
        rng = np.random.default_rng(rank)
        z = rng.integers(0, 1 << 64, size=(3, 17), dtype=np.uint64)
        t = torch.from_numpy(z.view(np.int64).copy())
        dp.allreduce(t)
        rows = dp.shard_rows(8)
        sess = types.SimpleNamespace(dp=dp, _replicated=0)
        off = TrioSession.shard_offset(sess, 40)
        sess._replicated = 1
        rep = TrioSession.shard_offset(sess, 40)
        q.put((rank, t.numpy().view(np.uint64).copy(), (rows.start, rows.stop), off, rep))
    finally:
        dist.destroy_process_group()


def test_gloo_allreduce_wraps_and_shards_partition():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    want = sum((np.random.default_rng(r).integers(0, 1 << 64, size=(3, 17), dtype=np.uint64) for r in range(world)),
               start=np.zeros((3, 17), np.uint64))
    for rank, t, rows, off, rep in res:
        assert np.array_equal(t, want)  # sum mod 2^64 on every rank
        assert rows == (rank * 4, rank * 4 + 4)
        assert off == (rank * 40, world * 40)
        assert rep == (0, 40)


def test_shard_rows_requires_divisible_batch():
    with pytest.raises(Exception):
        DataParallel(0, 3, None).shard_rows(8)


def _tp_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2104_10949_b200.engine import RssTensor
        from paper_2104_10949_b200.nn import TensorParallel

        tp = TensorParallel.from_process_group()
        full = np.arange(3 * 1 * 8 * 2 * 3, dtype=np.int64).reshape(3, 1, 8, 2, 3)
        sl = tp.slab(8)
        slab = RssTensor(torch.from_numpy(np.ascontiguousarray(full[:, :, sl])))
        got = tp.gather(slab).data.numpy()
        q.put((rank, np.array_equal(got, full), (sl.start, sl.stop)))
    finally:
        dist.destroy_process_group()


def test_gloo_tensor_parallel_gather_restores_channel_order():
    """TensorParallel (ResNet-50 b=1 output-channel slabs): the all-gather of
    per-rank channel slabs rebuilds the full (3, 1, C, H, W) activation."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_tp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for rank, ok, sl in res:
        assert ok
        assert sl == (rank * 4, rank * 4 + 4)
