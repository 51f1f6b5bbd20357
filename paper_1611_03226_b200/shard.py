"""Multi-GPU decomposition of the two workloads: independent
frame-range / block-range shards with one-frame / FIR-history halos,
exchanged point to point between neighbouring ranks -- no collective on
the data path.  The exchange helpers take torch tensors so the same code
runs over NCCL (CUDA tensors, the bench) and gloo (CPU tensors, tests)."""
from __future__ import annotations


def even_ranges(total: int, world: int, align: int = 1) -> list[tuple[int, int]]:
    """Contiguous [start, end) ranges, sizes multiples of `align` (except the last)."""
    units = -(-total // align)
    out = []
    for r in range(world):
        a = units * r // world * align
        b = min(total, units * (r + 1) // world * align)
        out.append((a, b))
    return out


def frame_shards(frames: int, world: int) -> list[tuple[int, int]]:
    return even_ranges(frames, world)


def block_shards(samples: int, period: int, world: int) -> list[tuple[int, int]]:
    """Sample ranges made of whole blocks (a block is one token)."""
    return even_ranges(samples, world, period)


def dpd_halo_block(schedule, first_block: int, branch: int) -> int | None:
    """Index of the last block before `first_block` in which `branch` is
    active (its tail is the branch's FIR history), or None (zero state).
    The schedule cycles per block (proj/src/dpd.cpp:208)."""
    for p in range(first_block - 1, -1, -1):
        if (int(schedule[p % len(schedule)]) >> (branch - 1)) & 1:
            return p
    return None


def exchange_tail(send_tail, recv_buf, rank: int, world: int):
    """Rank r sends `send_tail` (its last frame / last T-1 samples) to r+1 and
    receives r-1's into `recv_buf`.  Returns True if a halo was received."""
    import torch.distributed as dist
    staged = dist.get_backend() == "gloo" and (send_tail.is_cuda or recv_buf.is_cuda)
    if staged:  # gloo moves host memory only (functional checks of device runs)
        send_t, recv_t = send_tail.cpu(), recv_buf.new_empty(recv_buf.shape, device="cpu")
    else:
        send_t, recv_t = send_tail, recv_buf
    ops = []
    if rank + 1 < world:
        ops.append(dist.P2POp(dist.isend, send_t, rank + 1))
    if rank > 0:
        ops.append(dist.P2POp(dist.irecv, recv_t, rank - 1))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if staged and rank > 0:
        recv_buf.copy_(recv_t)
    return rank > 0


def dpd_halo_tails(schedule, ranges, period: int, taps: int, rank: int, peers: dict) -> list:
    """Per branch, a device pointer to the last T-1 raw samples of its last
    active block before this rank's block range -- wherever that block is:
    on the previous rank, or on any earlier one when the branch is gated off
    for whole shards (the frozen history of dpd.cpp:264-279) --
    or None (zero history).  ranges: every rank's [start, end) sample range;
    peers: rank -> base pointer of that rank's mapped shard (PeerBuffer)."""
    b0 = ranges[rank][0] // period
    out = []
    for b in range(1, 11):
        hb = dpd_halo_block(schedule, b0, b)
        if hb is None:
            out.append(None)
            continue
        owner = next(r for r, (s0, s1) in enumerate(ranges) if s0 // period <= hb < s1 // period)
        local = hb - ranges[owner][0] // period
        out.append(peers[owner] + 8 * ((local + 1) * period - (taps - 1)))
    return out


class PeerBuffer:
    """Rank r's views of the lower ranks' exported shard buffers (CUDA IPC):
    set up once (handles travel by all_gather_object -- setup, not the data
    path).  `ptr` / `device` are rank r-1's (the motion halo); `peers` maps
    every lower rank to its mapped base pointer (a DPD branch gated off for
    whole shards takes its FIR-history halo from further back).  Halos are
    pulled with copy-engine peer copies over NVLink (df_halo_copy) or read by
    the firing itself (df_dpd_fire_halo)."""

    def __init__(self, ptr: int, device: int, rank: int, world: int, lower: str = "all"):
        import ctypes as C

        import torch.distributed as dist

        from . import _lib
        n = _lib.lib().df_ipc_handle_size()
        h = (C.c_char * n)()
        _lib.call("df_ipc_get_handle", C.c_void_p(ptr), h)
        mine = (bytes(h), device)
        every = [None] * world
        dist.all_gather_object(every, mine)
        self.ptr = None
        self.device = None
        self.peers: dict[int, int] = {}
        self._mapped: list[int] = []
        wanted = range(rank) if lower == "all" else ([rank - 1] if rank > 0 else [])
        for r in wanted:
            handle, dev = every[r]
            hb = (C.c_char * n).from_buffer_copy(handle)
            p = C.c_void_p()
            _lib.call("df_ipc_open_handle", device, hb, C.byref(p))
            self.peers[r] = p.value
            self._mapped.append(p.value)
            if r == rank - 1:
                self.ptr, self.device = p.value, dev

    def close(self):
        from . import _lib
        for p in self._mapped:
            _lib.call("df_ipc_close_handle", __import__("ctypes").c_void_p(p))
        self._mapped = []
        self.peers = {}
        self.ptr = None
