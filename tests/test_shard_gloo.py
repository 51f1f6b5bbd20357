"""CPU, world size 2 over gloo: the shard + halo decomposition reproduces
the unsharded result exactly (the oracle stands in for the device kernels,
whose shard/halo parity is tested on the GPU in test_*_gpu.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1611_03226_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _motion_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, h, n = 40, 24, 10
    rgb = O.synth_bytes(n * w * h * 3, 77)
    f0, f1 = shard.frame_shards(n, world)[rank]
    fb = w * h * 3
    mine = torch.from_numpy(rgb[f0 * fb:f1 * fb].copy())
    halo = torch.empty(fb, dtype=torch.uint8)
    got_halo = shard.exchange_tail(mine[-fb:].clone(), halo, rank, world)
    out = O.motion_rgb(mine.numpy(), w, h, 32, halo.numpy() if got_halo else None)
    q.put((rank, out))
    dist.destroy_process_group()


def _dpd_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    period, blocks, T = 64, 12, 32
    x = O.synth_samples(period * blocks, 5)
    taps = O.random_taps(6, T)
    s0, s1 = shard.block_shards(period * blocks, period, world)[rank]
    mine = torch.from_numpy(x[2 * s0:2 * s1].copy())
    # static all-active schedule: the halo is the previous shard's last
    # T-1 raw samples (poly is recomputed from them)
    halo = torch.zeros(2 * period, dtype=torch.float32)
    tail = torch.zeros(2 * period, dtype=torch.float32)
    tail[-2 * (T - 1):] = mine[-2 * (T - 1):]
    got = shard.exchange_tail(tail, halo, rank, world)
    if got:  # oracle on [halo block, shard] from zero state, halo outputs dropped
        y = O.dpd(np.concatenate([halo.numpy(), mine.numpy()]), taps, [0x3FF], period)[2 * period:]
    else:
        y = O.dpd(mine.numpy(), taps, [0x3FF], period)
    q.put((rank, y))
    dist.destroy_process_group()


def _run(worker, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return np.concatenate([res[r] for r in range(world)])


def test_motion_frame_shards_with_halo_gloo():
    w, h, n = 40, 24, 10
    rgb = O.synth_bytes(n * w * h * 3, 77)
    np.testing.assert_array_equal(_run(_motion_worker), O.motion_rgb(rgb, w, h))


def test_dpd_block_shards_with_history_halo_gloo():
    period, blocks, T = 64, 12, 32
    x = O.synth_samples(period * blocks, 5)
    want = O.dpd(x, O.random_taps(6, T), [0x3FF], period)
    got = _run(_dpd_worker)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_ranges_and_halo_block_lookup():
    assert shard.frame_shards(300, 8)[0] == (0, 37) and shard.frame_shards(300, 8)[-1][1] == 300
    r = shard.block_shards(1 << 20, 4096, 3)
    assert all(a % 4096 == 0 for a, _ in r) and r[-1][1] == 1 << 20
    sched = [0b01, 0b10, 0b11]
    assert shard.dpd_halo_block(sched, 4, 1) == 3 and shard.dpd_halo_block(sched, 4, 2) == 2
    assert shard.dpd_halo_block(sched, 1, 2) is None
