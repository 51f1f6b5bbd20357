"""GPU, world sizes 2, 4 and 8 (processes on cuda:0, gloo for setup only):
the N>1 transport of bench.py -- each rank exports its shard buffer once
(CUDA IPC) and maps the lower ranks'; motion pulls its one-frame halo from
rank-1 with a copy-engine peer copy (df_halo_copy) and fires with
df_motion_fire_halo; DPD fires with df_dpd_fire_halo reading each branch's
FIR-history tail straight from whichever lower rank holds that branch's
last active block (a branch gated off for whole shards takes
its history from further back, dpd.cpp:264-279).  The concatenated shard
outputs must equal the oracle on the unsharded stream, byte for byte
(motion) and bit for bit (DPD).

Cases: small dynamic streams at world 2 and 4 (the 4-way one with a branch
gated off across two whole shards), BASELINE configs[3] (3840x2160 RGB,
40 frames, 8 frame-range shards) and the configs[4] structure (10 branches
x 32 taps, all active, 65536-sample blocks, 8 block-range shards) at 2^21
samples so the oracle stays fast."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.gpu

MOTION_CASES = {"small": (160, 48, 12, 4242), "4k": (3840, 2160, 40, 4343)}
DPD_CASES = {
    # period, blocks, T, input seed, schedule
    "dyn": (256, 24, 10, 31, [0x001, 0x3FF, 0x0F0, 0x2A5, 0x100, 0x003, 0x200]),
    # branch 10 only in block 2 (rank 0) and block 30 (rank 3): ranks 1..3
    # take its history from rank 0; branch 9 only in block 12 (rank 1).
    "gated": (128, 32, 10, 33, [0x003 | (0x200 if i in (2, 30) else 0) | (0x100 if i == 12 else 0) for i in range(32)]),
    "cfg5": (65536, 32, 32, 35, [0x3FF]),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _motion_worker(rank, world, port, q, case):
    from paper_1611_03226_b200 import _lib, device, motion, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, h, n, seed = MOTION_CASES[case]
        fb = w * h * 3
        rgb = O.synth_bytes(n * fb, seed)
        ranges = shard.frame_shards(n, world)
        f0, f1 = ranges[rank]
        mine = device.Buffer.from_array(rgb[f0 * fb:f1 * fb])
        dist.barrier()
        peer = shard.PeerBuffer(mine.ptr.value, 0, rank, world, lower="prev")
        actor = motion.MotionActor(w, h, motion.RGB, 32)
        out = device.Buffer((f1 - f0) * w * h)
        if rank > 0:
            halo = device.Buffer(fb)
            last = (ranges[rank - 1][1] - ranges[rank - 1][0] - 1) * fb
            _lib.call("df_halo_copy", 0, halo.ptr, peer.device, C.c_void_p(peer.ptr + last), fb, None)
            actor.fire_halo(halo, mine, out, f1 - f0)
        else:
            actor.fire(mine, out, f1 - f0)
        q.put((rank, out.download(np.uint8)))
        dist.barrier()  # every rank is done reading before anyone unmaps / frees
        peer.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _dpd_worker(rank, world, port, q, case):
    from paper_1611_03226_b200 import device, dpd, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        period, blocks, T, seed, sched = DPD_CASES[case]
        sched = np.array(sched, np.uint16)
        x = O.synth_samples(period * blocks, seed)
        taps = O.random_taps(seed + 1, T)
        ranges = shard.block_shards(period * blocks, period, world)
        s0, s1 = ranges[rank]
        b0, nb = s0 // period, (s1 - s0) // period
        mine = device.Buffer.from_array(x[2 * s0:2 * s1])
        ctrl = device.Buffer(4 * nb)
        dpd.config_tokens(sched, b0, nb, ctrl)  # global block indices: the schedule cycles per block
        dist.barrier()
        peer = shard.PeerBuffer(mine.ptr.value, 0, rank, world)  # maps every lower rank
        actor = dpd.DpdActor(period, taps)
        out = device.Buffer(8 * (s1 - s0))
        if rank > 0:
            tails = shard.dpd_halo_tails(sched, ranges, period, T, rank, peer.peers)
            actor.fire_halo(tails, ctrl, mine, out, nb)
        else:
            actor.fire(ctrl, mine, out, nb)
        actor.check()
        q.put((rank, out.download(np.float32)))
        dist.barrier()
        peer.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(worker, world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q, case)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return np.concatenate([got[r] for r in range(world)])


@pytest.mark.parametrize("case,world", [("small", 2), ("small", 4), ("4k", 8)])
def test_motion_frame_shards_ipc_halo(gpu, case, world):
    w, h, n, seed = MOTION_CASES[case]
    rgb = O.synth_bytes(n * w * h * 3, seed)
    want = O.motion_mt(rgb, w, h, 3, 32)
    got = _run(_motion_worker, world, case)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} bytes differ, first in frame {bad[0] // (w * h)}"


@pytest.mark.parametrize("case,world", [("dyn", 2), ("gated", 4), ("cfg5", 8)])
def test_dpd_block_shards_ipc_halo(gpu, case, world):
    period, blocks, T, seed, sched = DPD_CASES[case]
    x = O.synth_samples(period * blocks, seed)
    taps = O.random_taps(seed + 1, T)
    want = O.dpd_mt(x, taps, np.array(sched, np.uint16), period)
    got = _run(_dpd_worker, world, case)
    bad = np.nonzero(got.view(np.uint32) != want.view(np.uint32))[0]
    assert bad.size == 0, f"{bad.size} float words differ, first at sample {bad[0] // 2}"


def test_gated_case_needs_a_halo_beyond_the_neighbour():
    """The 'gated' schedule really exercises a halo from rank r-2 or
    earlier (checked on the host, no device needed for the arithmetic)."""
    from paper_1611_03226_b200 import shard
    period, blocks, T, _, sched = DPD_CASES["gated"]
    ranges = shard.block_shards(period * blocks, period, 4)
    peers = {0: 0, 1: 1 << 40, 2: 2 << 40}
    tails = shard.dpd_halo_tails(sched, ranges, period, T, 3, peers)
    assert tails[9] is not None and tails[9] < (1 << 40)  # branch 10 of rank 3 reads rank 0
    assert tails[8] is not None and (1 << 40) <= tails[8] < (2 << 40)  # branch 9 of rank 3 reads rank 1
