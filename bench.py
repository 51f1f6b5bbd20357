"""bench.py -- GPU-actor path of arXiv 1611.03226 (dynflow) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload motion720|motion4k|dpd1|dpd3|dpd5]

Default workload = BASELINE.json configs[1]: motion detection on 1280x720
RGB, 300 synthetic frames per GPU (frame-range sharded; one-frame halo from
the previous rank over NCCL P2P, no collective on the data path).  One
step = one firing of the fused motion actor over the rank's 300 frames.

--impl reference times the reference's own CPU implementation (the dynflow
network compiled from /root/reference into oracle/_ref, or the oracle port
when that is absent) on the box's host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
# Non-fused FP32 peak, MEASURED on the box (not in MEASURED_PEAKS.json):
# tools/ubench_ops.cu issued FMUL at 1106.0 and FADD at 1114.8 G warp-
# instructions/s on 148 SMs (profiles/r01_box_probe_and_pipe_ubench.log),
# i.e. 35.4 / 35.7 Top/s; the mean is the denominator.  The theoretical
# 148 x 128 x 1.965 GHz = 37.2 Top/s is reported beside it.
FP32_PEAK_TOPS = 32 * (1106.0 + 1114.8) / 2 / 1e3
FP32_PEAK_SOURCE = "measured (tools/ubench_ops FMUL/FADD, profiles/r01_box_probe_and_pipe_ubench.log)"
FP32_THEORETICAL_TOPS = 148 * 128 * 1.965e9 / 1e12


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


WORKLOADS = {
    # name: (kind, params)
    "motion720": ("motion", dict(w=1280, h=720, frames=300, fmt=3, thr=32,
                                 label="Motion detection 1280x720 RGB, 300 synthetic frames per GPU")),
    # The reference's own input format (8-bit gray, proj/include/dynflow/motion.hpp:11-16).
    "motion720gray": ("motion", dict(w=1280, h=720, frames=300, fmt=1, thr=32,
                                     label="Motion detection 1280x720 gray (reference format), 300 frames per GPU")),
    "motion4k": ("motion", dict(w=3840, h=2160, frames=40, fmt=3, thr=32,
                                label="Motion detection 3840x2160 RGB, 40 frames per GPU (320 at 8 GPUs)")),
    "dpd1": ("dpd", dict(samples=1 << 20, period=65536, T=10, sched="first2",
                         label="DPD 2 branches x 10-tap, 2^20 samples, fixed config")),
    "dpd3": ("dpd", dict(samples=1 << 26, period=4096, T=10, sched="ramp",
                         label="DPD dynamic 1->10 branches per 4096-sample block (ramp), 2^26 samples")),
    "dpd5": ("dpd", dict(samples=1 << 27, period=65536, T=32, sched="all10",
                         label="DPD 10 branches x 32-tap, 2^27 samples per GPU (2^30 at 8 GPUs)")),
}


# ------------------------------------------------------------------ helpers
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and BACKEND == "gloo":
        # Functional check of the N>1 path on a box with fewer GPUs than
        # ranks (gloo cannot see CUDA memory; halos are staged on the host).
        import torch
        local %= max(1, torch.cuda.device_count())
    return rank, world, local


# L2 flush buffer: > 126 MB L2 (B200); also the threshold below which a
# workload's in+out bytes need a flush between timed steps.
L2_FLUSH_BYTES = 256 << 20

# Process-group backend: NCCL for every measured run; DF_BENCH_BACKEND=gloo
# only for functional checks of the multi-rank path.
BACKEND = os.environ.get("DF_BENCH_BACKEND", "nccl")
# Halo transport at N>1: "ipc" (default) -- rank r maps rank r-1's shard
# buffer once (CUDA IPC) and pulls each step's halo with a copy-engine peer
# copy over NVLink on a side stream, overlapped with the previous step's
# kernel; "p2p" -- NCCL send/recv on the compute stream.
HALO = os.environ.get("DF_BENCH_HALO", "ipc")


class HaloPipe:
    """Double-buffered halo pulls on a side stream (peer copies
    overlapped with interior work).  pull(i, copies) issues step i's copies
    [(dst_ptr, src_ptr, bytes)] into slot i % 2 and makes `stream` wait for
    them; release(slot) marks the slot consumed (after its consumer kernel)."""

    def __init__(self, torch, stream, local, peer_device):
        self.torch, self.stream, self.local, self.peer = torch, stream, local, peer_device
        self.hs = torch.cuda.Stream()
        self.ready = [torch.cuda.Event(), torch.cuda.Event()]
        self.free = [torch.cuda.Event(), torch.cuda.Event()]
        self.used = [False, False]

    def pull(self, i, copies):
        from paper_1611_03226_b200 import _lib
        k = i % 2
        with self.torch.cuda.stream(self.hs):
            if self.used[k]:
                self.hs.wait_event(self.free[k])
            hsh = C.c_void_p(self.hs.cuda_stream)
            for dst, src, nbytes in copies:
                _lib.call("df_halo_copy", self.local, C.c_void_p(dst), self.peer, C.c_void_p(src), nbytes, hsh)
            self.ready[k].record(self.hs)
        self.stream.wait_event(self.ready[k])
        return k

    def release(self, k):
        self.free[k].record(self.stream)
        self.used[k] = True


def traffic_from_profiles(kernel: str, workload: str):
    """dram bytes per launch from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    return d.get(workload, {}).get(kernel)


# ------------------------------------------------------------------ ours
def bench_motion_ours(args, p, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_1611_03226_b200 import _lib, device, motion, shard

    _lib.require_gpu()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    W, H, F, fmt = p["w"], p["h"], p["frames"], p["fmt"]
    in_frame, out_frame = W * H * fmt, W * H
    stream = torch.cuda.current_stream()
    sh = C.c_void_p(stream.cuda_stream)
    inp_buf = device.Buffer(F * in_frame, local)  # cudaMalloc'ed: exportable to the neighbour rank
    inp = inp_buf.as_tensor()
    out = torch.empty(F * out_frame, dtype=torch.uint8, device=dev)
    halos = [torch.empty(in_frame, dtype=torch.uint8, device=dev) for _ in range(2)]
    _lib.call("df_fill_random_u8", C.c_void_p(inp.data_ptr()), inp.numel(), 1234 + rank, sh)
    actor = motion.MotionActor(W, H, fmt, p["thr"], device=local)
    peer = pipe = None
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()  # every shard is filled before a neighbour maps it
        if HALO == "ipc":
            peer = shard.PeerBuffer(inp.data_ptr(), local, rank, world, lower="prev")
            if rank > 0:
                pipe = HaloPipe(torch, stream, local, peer.device)
    nstep = [0]

    def step(ev_k0=None, ev_k1=None):
        sh = C.c_void_p(torch.cuda.current_stream().cuda_stream)  # the capture stream inside a graph
        k = 0
        if world > 1:
            # One-frame halo: the previous rank's last input frame.
            if pipe is not None:
                k = pipe.pull(nstep[0], [(halos[nstep[0] % 2].data_ptr(), peer.ptr + (F - 1) * in_frame,
                                          in_frame)])
            elif HALO != "ipc":
                shard.exchange_tail(inp[(F - 1) * in_frame:], halos[0], rank, world)
        nstep[0] += 1
        if rank == 0:
            _lib.call("df_motion_set_prev_frame", actor.handle, None, sh)  # black initial token
        if ev_k0 is not None:
            ev_k0.record(stream)
        if rank > 0:
            # gauss(halo) is computed inside the firing (no separate pass)
            _lib.call("df_motion_fire_halo", actor.handle, C.c_void_p(halos[k].data_ptr()),
                      C.c_void_p(inp.data_ptr()), C.c_void_p(out.data_ptr()), F, sh)
            if pipe is not None:
                pipe.release(k)
        else:
            _lib.call("df_motion_fire", actor.handle, C.c_void_p(inp.data_ptr()), C.c_void_p(out.data_ptr()), F,
                      sh)
        if ev_k1 is not None:
            ev_k1.record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    graph = None
    launches0 = device.kernel_launches()
    if world == 1:
        # The K timed steps are captured in ONE CUDA graph so host-side
        # enqueue latency never starves the device between steps; it is
        # replayed once untimed first (warm-up that also keeps the device
        # busy while the timed replay is submitted).
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(args.steps):
                step()
        torch.cuda.synchronize()
    launches = device.kernel_launches() - launches0
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        if graph is not None:
            graph.replay()
        t0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(args.steps):
                step(*kev[i])
        t1.record(stream)
        torch.cuda.synchronize()
    if graph is None:
        launches = device.kernel_launches() - launches0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    # at N=1 the fused kernel is the whole step (plus a delay-token memset)
    kms = ms if graph is not None else statistics.mean(a.elapsed_time(b) for a, b in kev)
    ms, kms = max_over_ranks(ms, world), max_over_ranks(kms, world)

    # e2e through the C-ABI host-buffer call: pinned H2D + fire + D2H per step.
    hin = device.PinnedArray(F * in_frame, np.uint8)
    hout = device.PinnedArray(F * out_frame, np.uint8)
    hin.array[:] = np.frombuffer(np.random.default_rng(rank).bytes(F * in_frame), np.uint8)
    actor.run_host(hin.array, hout.array)  # warm
    e2e_t = []
    for _ in range(max(2, min(args.steps, 5))):
        torch.cuda.synchronize()
        a = time.perf_counter()
        actor.run_host(hin.array, hout.array)
        e2e_t.append(time.perf_counter() - a)
    e2e_s = max_over_ranks(statistics.median(e2e_t), world)
    torch.cuda.synchronize()
    if peer is not None:  # unmap the neighbour's shard before anyone frees theirs
        peer.close()
        dist.barrier()

    value = world * F / (ms / 1e3)
    bytes_alg = 4.0 * W * H * F if fmt == 3 else 2.0 * W * H * F
    achieved = bytes_alg / (kms / 1e3) / 1e9
    hbm, hbm_src = peaks()
    kname = actor.kernel_name
    traffic = traffic_from_profiles(kname, args.workload)
    res = {
        "metric": "motion-detect frames/s",
        "value": round(value, 1),
        "unit": "frames/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (device splitmix64 bytes; " + ("RGB interleaved)" if fmt == 3 else "8-bit gray)"),
        "config": {"workload": p["label"], "width": W, "height": H, "frames_per_gpu": F,
                   "threshold": p["thr"], "input": "rgb" if fmt == 3 else "gray",
                   "chain": "gray->gauss5x5->|cur-prev|>thr->median5 (reference-pinned)",
                   "parallelism": f"frame-range shards x{world}, 1-frame halo via "
                                  + ("NVLink peer copy (CUDA IPC), overlapped" if HALO == "ipc" else "NCCL P2P"),
                   "l2": f"inputs {F * in_frame / 1e6:.0f} MB per GPU > 126 MB L2 (no flush needed)"},
        "e2e": {"value": round(world * F / e2e_s, 1), "unit": "frames/s",
                "h2d_bytes_per_step": F * in_frame, "d2h_bytes_per_step": F * out_frame,
                "path": "df_motion_run_host (C ABI, pinned host buffers, chunked H2D/fire/D2H)"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "kernel": kname, "kernel_ms": round(kms, 4),
                     "algorithmic_bytes_per_launch": bytes_alg, "peak_source": hbm_src},
        "clocks": clk.summary(),
    }
    return res


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if BACKEND == "gloo" else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dpd_schedule(kind: str, blocks: int) -> np.ndarray:
    if kind == "first2":
        return np.array([0b11], np.uint16)
    if kind == "all10":
        return np.array([0x3FF], np.uint16)
    if kind == "ramp":
        return np.array([(1 << (1 + i % 10)) - 1 for i in range(10)], np.uint16)
    raise ValueError(kind)


def dpd_flops_per_sample(sched: np.ndarray, T: int) -> float:
    # B*(8T+4) + B_max + 3 per sample (+1 sqrt), mean over the schedule
    tot = 0.0
    for m in sched:
        B = bin(int(m)).count("1")
        bmax = int(m).bit_length()
        tot += B * (8 * T + 4) + bmax + 3
    return tot / len(sched)


def bench_dpd_ours(args, p, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_1611_03226_b200 import _lib, device, dpd

    _lib.require_gpu()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    N, period, T = p["samples"], p["period"], p["T"]
    blocks = N // period
    sched = dpd_schedule(p["sched"], blocks)
    stream = torch.cuda.current_stream()
    sh = C.c_void_p(stream.cuda_stream)
    # Input + output smaller than L2 (DPD-1: 16 MB vs 126 MB): consecutive
    # steps fire on a rotating pool of R input/output batches whose total
    # exceeds L2, so every step reads a batch last touched R-1 steps
    # (>= 256 MB of traffic) earlier -- cold, as a streaming actor sees it --
    # and K steps run back to back between one event pair (per-step event
    # pairs around a flushed step add ~6 us of event-node overhead to a
    # ~12 us firing: tools/probe_event_overhead.py, profiles/r02_dpd_timing.txt).
    R = max(1, -(-L2_FLUSH_BYTES // (16 * N)))
    x_buf = device.Buffer(8 * N * R, local)  # cudaMalloc'ed: exportable to the neighbour rank
    x_pool = x_buf.as_tensor(np.float32)
    y_pool = torch.empty(2 * N * R, dtype=torch.float32, device=dev)
    x, y = x_pool[: 2 * N], y_pool[: 2 * N]
    ctrl = torch.empty(blocks, dtype=torch.int32, device=dev)
    _lib.call("df_fill_random_pm1", C.c_void_p(x_pool.data_ptr()), 2 * N * R, 99 + rank, sh)
    taps = np.random.default_rng(808).uniform(-0.5, 0.5, size=(10, T, 2)).astype(np.float32)
    actor = dpd.DpdActor(period, taps, device=local)
    sched_np = np.ascontiguousarray(sched)
    # Rank r holds global blocks [r*blocks, (r+1)*blocks): its control tokens
    # continue the global schedule (dpd.cpp:208 schedule[firing % len]).
    _lib.call("df_dpd_config_tokens", local, sched_np.ctypes.data_as(C.c_void_p), sched_np.size, rank * blocks,
              blocks, C.c_void_p(ctrl.data_ptr()), sh)

    # Block-range shard of a weak-scaled stream: rank r holds blocks
    # [r*blocks, (r+1)*blocks).  FIR-history halo: for each branch, the last
    # T-1 samples of its last active block in the previous rank's range
    # (read in-kernel from the neighbour's mapped shard, or NCCL P2P; no
    # collective); rank 0 starts from zero history.
    from paper_1611_03226_b200 import shard
    H1 = max(T - 1, 1)
    tails = torch.zeros(10 * H1 * 2, dtype=torch.float32, device=dev)
    halo = torch.zeros_like(tails)
    tail_src = []
    for b in range(1, 11):  # last active block of this rank's range (local index), for the P2P variant
        hb = shard.dpd_halo_block(sched, (rank + 1) * blocks, b)
        tail_src.append(hb - rank * blocks if hb is not None and hb >= rank * blocks else None)
    peer = None
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()  # every shard is filled before a neighbour maps it
        if HALO == "ipc":
            peer = shard.PeerBuffer(x.data_ptr(), local, rank, world)
    # IPC: the firing reads each branch's halo tail straight from the
    # neighbour's mapped shard over NVLink (df_dpd_fire_halo) -- no copy, no
    # extra launch; only the block-start tiles that need a tail touch it.
    tail_ptrs = None
    if peer is not None and rank > 0:
        # The global stream is the ranks' shards back to back (the schedule
        # cycling over global block indices), so each branch's halo is
        # the tail of its last active block before this shard, on whichever
        # lower rank holds it (shard.dpd_halo_tails).  Pool slot k of every
        # rank holds the same step, so slot k's tails sit k*8N bytes further.
        ranges = [(r * N, (r + 1) * N) for r in range(world)]
        tails_g = shard.dpd_halo_tails(sched, ranges, period, T, rank, peer.peers)  # global block indices
        tail_ptrs = [(C.c_void_p * 10)(*[C.c_void_p(t + 8 * N * k) if t is not None else None for t in tails_g])
                     for k in range(R)]

    def step(i=0):
        sh = C.c_void_p(torch.cuda.current_stream().cuda_stream)  # the capture stream inside a graph
        k = i % R
        xk, yk = x_pool[2 * N * k: 2 * N * (k + 1)], y_pool[2 * N * k: 2 * N * (k + 1)]
        if world > 1 and HALO != "ipc":  # NCCL P2P variant: exchange the tails, set the histories
            for b, hb in enumerate(tail_src):
                if hb is not None:
                    a0 = 2 * ((hb + 1) * period - H1)
                    tails[2 * H1 * b: 2 * H1 * (b + 1)].copy_(xk[a0: a0 + 2 * H1])
            if shard.exchange_tail(tails, halo, rank, world):
                for b in range(10):
                    _lib.call("df_dpd_set_history", actor.handle, C.c_void_p(halo.data_ptr() + 8 * H1 * b), H1,
                              1 << b, sh)
        if tail_ptrs is not None:
            _lib.call("df_dpd_fire_halo", actor.handle, tail_ptrs[k], C.c_void_p(ctrl.data_ptr()),
                      C.c_void_p(xk.data_ptr()), C.c_void_p(yk.data_ptr()), blocks, sh)
        else:
            _lib.call("df_dpd_fire", actor.handle, C.c_void_p(ctrl.data_ptr()), C.c_void_p(xk.data_ptr()),
                      C.c_void_p(yk.data_ptr()), blocks, sh)

    # Warm-up walks the whole pool once (first touch of every batch).
    for i in range(max(args.warmup, R)):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    graph = lead = None
    if world == 1 or HALO == "ipc":
        # K steps, one graph (see bench_motion_ours).  At N > 1 the IPC
        # transport needs no per-step communication (the firing reads its
        # halo over NVLink), so the steps are pure launches and capture too.
        # `lead` is K untimed steps replayed just before the timed graph so
        # the device is busy while the timed graph is submitted; the timed
        # steps continue the pool rotation after it (steps K..2K-1).
        lead = torch.cuda.CUDAGraph()
        with torch.cuda.graph(lead):
            for i in range(args.steps):
                step(i)
        launches0 = device.kernel_launches()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for i in range(args.steps, 2 * args.steps):
                step(i)
        launches = device.kernel_launches() - launches0
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    else:
        launches0 = device.kernel_launches()
    with ClockSampler(local) as clk:
        if lead is not None:
            lead.replay()
        t0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(args.steps, 2 * args.steps):
                step(i)
        t1.record(stream)
        torch.cuda.synchronize()
    if graph is None:
        launches = device.kernel_launches() - launches0
    ms = max_over_ranks(t0.elapsed_time(t1) / args.steps, world)
    kms = ms
    actor.check()
    kname = actor.kernel_name  # the timed firings' main kernel (before run_host's chunked firings)

    hin = device.PinnedArray(2 * N, np.float32)
    hout = device.PinnedArray(2 * N, np.float32)
    hin.array[:] = np.random.default_rng(rank).uniform(-1, 1, 2 * N).astype(np.float32)
    actor.run_host(hin.array, hout.array, sched)
    e2e_t = []
    for _ in range(max(2, min(args.steps, 5))):
        a = time.perf_counter()
        actor.run_host(hin.array, hout.array, sched)
        e2e_t.append(time.perf_counter() - a)
    e2e_s = max_over_ranks(statistics.median(e2e_t), world)
    if peer is not None:  # unmap the neighbour's shard before anyone frees theirs
        torch.cuda.synchronize()
        peer.close()
        dist.barrier()

    fps = dpd_flops_per_sample(sched, T)
    achieved_tops = N * fps / (kms / 1e3) / 1e12
    hbm, _ = peaks()
    return {
        "metric": "DPD Msamples/s",
        "value": round(world * N / (ms / 1e3) / 1e6, 1),
        "unit": "Msamples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (device uniform[-1,1) complex samples)",
        "config": {"workload": p["label"], "samples_per_gpu": N, "period": period, "taps_per_branch": T,
                   "schedule": p["sched"],
                   "parallelism": f"block-range shards x{world}, per-branch FIR-history halo via "
                                  + ("in-kernel NVLink peer reads (CUDA IPC)" if HALO == "ipc" else "NCCL P2P"),
                   "l2": f"in+out {16 * N / 1e6:.0f} MB per GPU"
                         + (f" < L2: steps rotate over {R} input/output batches ({16 * N * R >> 20} MB > 126 MB L2), "
                            "so every step's input is cold; K steps back to back, one event pair"
                            if R > 1 else " > 126 MB L2 (no flush needed)")},
        "e2e": {"value": round(world * N / e2e_s / 1e6, 1), "unit": "Msamples/s",
                "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N,
                "path": "df_dpd_run_host (C ABI, pinned host buffers)"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "fp32", "achieved": round(achieved_tops, 2), "peak": round(FP32_PEAK_TOPS, 2),
                     "unit": "Top/s (non-fused FP32)", "frac": round(achieved_tops / FP32_PEAK_TOPS, 4),
                     "peak_source": FP32_PEAK_SOURCE,
                     "frac_of_theoretical": round(achieved_tops / FP32_THEORETICAL_TOPS, 4),
                     "traffic": traffic_from_profiles(kname, args.workload),
                     "kernel": kname, "kernel_ms": round(kms, 4), "flops_per_sample": fps,
                     "hbm_frac": round(16 * N / (kms / 1e3) / 1e9 / hbm, 4)},
        "clocks": clk.summary(),
    }


# ------------------------------------------------------------------ CPU
def cpu_motion(p, steps, warmup, nets=None):
    """The reference's own dynflow motion network (5 actor threads,
    proj/src/motion.cpp:107-218) on the FULL configuration: one step is all
    of the workload's frames (300 at 720p), split into `nets` contiguous
    frame ranges run as concurrent networks to use the host's cores (the
    frame-range sharding our multi-GPU path uses).  value = the reference's
    own metric, frames / active_seconds("sink") (proj/src/bench.cpp:
    341-347), with the sink-active window of concurrent networks taken as
    the longest one; median over steps.  Wall time per step (network build,
    thread spawn, fill and drain included) is reported beside it.  RGB input
    is converted to gray before the run (the reference takes gray frames).
    Falls back to the single-thread oracle port without oracle/_ref."""
    from oracle import oracle as O
    W, H, F = p["w"], p["h"], p["frames"]
    rgb_in = p.get("fmt", 3) == 3
    ncpu = len(os.sched_getaffinity(0))
    if O.ref_available():
        R = O.ref()
        # 8 networks on the 16-core box: gauss and med are the two busy actor
        # threads of a network (3 / 5 / 8 networks: 177 / 281 / 392 frames/s,
        # profiles/r02_cpu_baseline_probe.txt).
        nets = nets or int(os.environ.get("DF_CPU_NETS", "0")) or max(1, ncpu // 2)
        frames_in = O.synth_bytes(F * W * H * (3 if rgb_in else 1), 5)
        gray = O.rgb_to_gray(frames_in) if rgb_in else frames_in
        ranges = [(F * i // nets, F * (i + 1) // nets) for i in range(nets)]
        out = np.empty(F * W * H, np.uint8)
        act = [0.0] * nets

        def one(i):
            f0, f1 = ranges[i]
            a, w_ = C.c_double(), C.c_double()
            rc = R.ref_motion_network(gray[f0 * W * H:].ctypes.data_as(C.c_void_p), f1 - f0, W, H, 32, 1,
                                      out[f0 * W * H:].ctypes.data_as(C.c_void_p), C.byref(a), C.byref(w_))
            assert rc == 0
            act[i] = a.value

        active, wall = [], []
        for s in range(warmup + steps):
            ts = [threading.Thread(target=one, args=(i,)) for i in range(nets)]
            a = time.perf_counter()
            for t in ts:
                t.start()
            for t in ts:
                t.join()
            if s >= warmup:
                wall.append(time.perf_counter() - a)
                active.append(max(act))
        return {"value": round(F / statistics.median(active), 2), "unit": "frames/s",
                "cores": min(ncpu, 5 * nets), "kind": "reference",
                "wall_value": round(F / statistics.median(wall), 2),
                "sample": f"full config: {F} frames {W}x{H} per step as {nets} concurrent dynflow motion networks "
                          f"(5 actor threads each) on contiguous frame ranges"
                          + (", gray(RGB) conversion outside the timed runs" if rgb_in else " (gray)")
                          + f"; value = frames / sink-active seconds (bench.cpp:341-347, longest of the {nets}), "
                            f"wall_value = frames / step wall time; median of {steps}"}
    n = 4
    frames_in = O.synth_bytes(n * W * H * (3 if rgb_in else 1), 5)
    a = time.perf_counter()
    (O.motion_rgb if rgb_in else O.motion_gray)(frames_in, W, H)
    t = time.perf_counter() - a
    return {"value": round(n / t, 2), "unit": "frames/s", "cores": 1, "kind": "port",
            "sample": f"oracle port, {n} frames {W}x{H} {'RGB' if rgb_in else 'gray'}, 1 thread"}


def cpu_dpd(p, steps, warmup):
    """CPU reference for a DPD config, timed on this host's cores.

    - k >= 2 masks, T = 10: the reference's own network (15 actor threads),
      cmd_dpd's method.
    - k = 1 masks, T = 10: the network rejects them (check_config); the
      reference's single-thread oracle_dpd runs them.  One instance per
      host core on its own copy of the sample (ctypes drops the GIL).
    - T != 10 (the reference is fixed at 10 taps): the C oracle port, one
      instance per host core likewise.
    """
    from oracle import oracle as O
    period, T = p["period"], p["T"]
    n = min(p["samples"], max(period, 1 << 20))
    n -= n % period
    sched = dpd_schedule(p["sched"], n // period)
    x = O.synth_samples(n, 810)
    taps = O.random_taps(808, T)
    ncpu = len(os.sched_getaffinity(0))
    use_ref = O.ref_available() and T == 10 and all(bin(int(m)).count("1") >= 2 for m in sched)
    use_ref_oracle = O.ref_available() and T == 10 and not use_ref
    sc = np.ascontiguousarray(sched)
    workers = 1 if use_ref else ncpu
    outs = [np.empty_like(x) for _ in range(workers)]

    def one(i):
        if use_ref_oracle:
            rc = O.ref().ref_oracle_dpd(x.ctypes.data_as(C.c_void_p), n, taps.ctypes.data_as(C.c_void_p),
                                        sc.ctypes.data_as(C.c_void_p), sc.size, period,
                                        outs[i].ctypes.data_as(C.c_void_p))
            assert rc == 0
        else:
            O.dpd(x, taps, sched, period)

    times, walls = [], []
    reps = max(steps, 5) if use_ref else steps  # cmd_dpd: median of 5 reps (bench.cpp:391-397)
    for s in range(warmup + reps):
        if use_ref:
            R = O.ref()
            a_, w_ = C.c_double(), C.c_double()
            a = time.perf_counter()
            rc = R.ref_dpd_network(x.ctypes.data_as(C.c_void_p), n, taps.ctypes.data_as(C.c_void_p),
                                   sc.ctypes.data_as(C.c_void_p), sc.size, period, outs[0].ctypes.data_as(C.c_void_p),
                                   C.byref(a_), C.byref(w_))
            assert rc == 0
            if s >= warmup:
                walls.append(time.perf_counter() - a)
            el = a_.value  # the reference's metric: samples / active_seconds("sink")
        else:
            ts = [threading.Thread(target=one, args=(i,)) for i in range(workers)]
            a = time.perf_counter()
            for t_ in ts:
                t_.start()
            for t_ in ts:
                t_.join()
            el = time.perf_counter() - a
        if s >= warmup:
            times.append(el)
    t = statistics.median(times)
    if use_ref:
        full = n == p["samples"]
        return {"value": round(n / t / 1e6, 2), "unit": "Msamples/s", "cores": min(ncpu, 15), "kind": "reference",
                "wall_value": round(n / statistics.median(walls) / 1e6, 2),
                "sample": f"{'full config: ' if full else ''}dynflow DPD network (15 actor threads), {n} samples, "
                          f"period {period}; value = samples / sink-active seconds (cmd_dpd, bench.cpp:391-397), "
                          f"wall_value = samples / run() wall time; median of {reps}"}
    if use_ref_oracle:
        return {"value": round(workers * n / t / 1e6, 2), "unit": "Msamples/s", "cores": workers,
                "kind": "reference",
                "sample": f"dynflow oracle_dpd (the network rejects k=1 masks) x {workers} concurrent instances, "
                          f"{n} samples each, period {period}; median of {steps}"}
    return {"value": round(workers * n / t / 1e6, 2), "unit": "Msamples/s", "cores": workers, "kind": "port",
            "sample": f"oracle port (the reference is fixed at 10 taps, T={T}) x {workers} concurrent instances, "
                      f"{n} samples each; median of {steps}"}


# ------------------------------------------------------------------ networks
def _timed_steps(step, steps, warmup, stream):
    from paper_1611_03226_b200 import device
    for _ in range(warmup):
        step()
    stream.synchronize()
    e0, e1 = device.Event(), device.Event()
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_ms(e1) / steps


def motion_network(p, steps, warmup):
    """The motion actor inside its network on device channels: source ->
    motion (input channel at rate F, rate-1 self-loop delay channel with the
    black initial token, proj/src/motion.cpp:131) -> sink.  The source's
    frames are resident in the input channel's storage (both Eq. 1 halves);
    each step commits the source's write, fires the actor on the regions it
    resolves on the device, and commits the sink's read (1-thread kernels)."""
    from paper_1611_03226_b200 import _lib, device, motion
    from paper_1611_03226_b200.channel import DeviceChannel
    W, H, F, fmt = p["w"], p["h"], p["frames"], p["fmt"]
    s = device.Stream()
    cin = DeviceChannel(W * H * fmt, F)
    cout = DeviceChannel(W * H, F)
    delay = DeviceChannel(W * H, 1, has_delay=True, initial_token=np.zeros(W * H, np.uint8))
    _lib.call("df_fill_random_u8", C.c_void_p(_lib.lib().df_channel_storage(cin.handle)), cin.capacity_bytes, 77,
              s.handle)
    a = motion.MotionActor(W, H, fmt, p["thr"])

    def step():
        wr = cin.write_start(F)
        cin.write_end(wr, s)
        a.fire_channels(cin, delay, cout, s)
        rd = cout.read_start(F)
        cout.read_end(rd, s)

    ms = _timed_steps(step, steps, warmup, s)
    for ch in (cin, cout, delay):
        ch.check()
    hbm, _ = peaks()
    bytes_alg = (4.0 if fmt == 3 else 2.0) * W * H * F
    return {"value": round(F / (ms / 1e3), 1), "unit": "frames/s", "ms_per_step": round(ms, 4),
            "roofline_frac": round(bytes_alg / (ms / 1e3) / 1e9 / hbm, 4), "roofline_bound": "hbm",
            "path": "source -> motion (device channels: Eq. 1 input/output rings at rate F, Fig. 2 delay "
                    "self-loop; regions and commits on the device) -> sink; host-endpoint commits are 1-thread "
                    "kernels; 3 launches per step"}


def dpd_network(p, steps, warmup):
    """The dynamic DPD actor inside its network on device channels: config
    -> ctrl channel (4-byte control tokens, one per block) and source -> in
    channel -> DPD (consumes K control tokens on the device) -> out channel
    -> sink.  Tokens and samples are resident in both Eq. 1 halves."""
    from paper_1611_03226_b200 import _lib, device, dpd
    from paper_1611_03226_b200.channel import DeviceChannel
    N, period, T = p["samples"], p["period"], p["T"]
    K = N // period
    sched = np.ascontiguousarray(dpd_schedule(p["sched"], K))
    s = device.Stream()
    cctl = DeviceChannel(4, K)
    cin = DeviceChannel(8 * period, K)
    cout = DeviceChannel(8 * period, K)
    L = _lib.lib()
    _lib.call("df_fill_random_pm1", C.c_void_p(L.df_channel_storage(cin.handle)), cin.capacity_bytes // 4, 99,
              s.handle)
    for half in range(cctl.capacity_tokens // K):
        _lib.call("df_dpd_config_tokens", 0, sched.ctypes.data_as(C.c_void_p), sched.size, 0, K,
                  C.c_void_p(L.df_channel_storage(cctl.handle) + 4 * K * half), s.handle)
    taps = np.random.default_rng(808).uniform(-0.5, 0.5, size=(10, T, 2)).astype(np.float32)
    a = dpd.DpdActor(period, taps)

    def step():
        for ch in (cctl, cin):
            wr = ch.write_start(K)
            ch.write_end(wr, s)
        a.fire_channels(cctl, cin, cout, K, s)
        rd = cout.read_start(K)
        cout.read_end(rd, s)

    ms = _timed_steps(step, steps, warmup, s)
    a.check()
    for ch in (cctl, cin, cout):
        ch.check()
    flops = dpd_flops_per_sample(sched, T) * N
    return {"value": round(N / (ms / 1e3) / 1e6, 1), "unit": "Msamples/s", "ms_per_step": round(ms, 4),
            "roofline_frac": round(flops / (ms / 1e3) / 1e12 / FP32_PEAK_TOPS, 4), "roofline_bound": "fp32",
            "path": "config -> ctrl channel, source -> in channel -> dpd (control tokens consumed on the device) "
                    "-> out channel -> sink; host-endpoint commits are 1-thread kernels"}


def resident_networks():
    """The reference's own network shapes (15-actor DPD, 5-actor motion with
    its delay channel) as device-resident actors -- one persistent kernel,
    control tokens dispatched per firing on the device (dfh_*_run_resident)
    -- measured by the reference's metric (units / active_seconds("sink")).
    DPD-1's full configuration; motion 1280x720 x 300 in the reference's
    gray format (that network has no RGB front end)."""
    from paper_1611_03226_b200 import host_api as H
    # Inputs from the library's copies of the reference's generators
    # (dfh_synth; the same streams as synth_samples / random_taps /
    # synth_frames, proj/src/dpd.cpp:467-505, motion.cpp:254-260).
    x = H.synth("samples", 1 << 20, 810)
    taps = H.synth("taps", 10, 808).reshape(10, 10, 2)
    H.dpd_run_resident(x, taps, [3], 65536, branch_ctas=32)
    ms = [H.dpd_run_resident(x, taps, [3], 65536, branch_ctas=32)[1] for _ in range(3)]
    f = H.synth("frames", 300 * 1280 * 720, 5)
    mm = [H.motion_run_resident(f, 1280, 720, 32, ctas=96)[1] for _ in range(2)]
    mr = [H.motion_run_resident(f, 1280, 720, 32, rate=10, ctas=96)[1] for _ in range(2)]
    return {"dpd1": {"value": round((1 << 20) / (statistics.median(ms) / 1e3) / 1e6, 1), "unit": "Msamples/s",
                     "path": "dfh_dpd_run_resident: source, config, split, 10 branches, adder, sink (56 channels), "
                             "32 CTAs per branch"},
            "motion720gray": {"value": round(300 / (statistics.median(mm) / 1e3), 1), "unit": "frames/s",
                              "path": "dfh_motion_run_resident: source, gauss, thres, med, sink with the "
                                      "gauss_thres_prev delay channel, 480 CTAs shared by work (gauss 160, med 120, thres 80, source / sink 60)"},
            "motion720gray_rate10": {"value": round(300 / (statistics.median(mr) / 1e3), 1), "unit": "frames/s",
                                     "path": "the same network at token rate 10 (10 frames per token: the reference's "
                                             "--rate option, bench.cpp:212)"},
            "metric": "units / sink-active seconds (bench.cpp:341-347, :391-397), device timestamps"}


def bench_reference(args, kind, p, rank, world):
    if rank != 0:
        return None
    if kind == "motion":
        cb = cpu_motion(p, args.steps, args.warmup)
        metric, unit = "motion-detect frames/s", "frames/s"
    else:
        cb = cpu_dpd(p, args.steps, args.warmup)
        metric, unit = "DPD Msamples/s", "Msamples/s"
    return {"impl": "reference", "metric": metric, "value": cb["value"], "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8" if kind == "motion" else "f32", "data": "synthetic",
            "config": {"workload": p["label"]}, "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="motion720", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the DPD configs reported beside the headline at N=1")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local = dist_env()
    kind, p = WORKLOADS[args.workload]

    if args.impl == "reference":
        res = bench_reference(args, kind, p, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if BACKEND == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # One line per rank on stderr (the JSON line stays rank 0's only).
        print(f"bench: rank {rank}/{world} on cuda:{local} ({torch.cuda.get_device_name(local)}), "
              f"process group {dist.get_backend()}, halo transport {HALO}", file=sys.stderr, flush=True)
    res = (bench_motion_ours if kind == "motion" else bench_dpd_ours)(args, p, rank, world, local)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = (cpu_motion(p, 3, 1) if kind == "motion" else cpu_dpd(p, 3, 1))
        if world == 1 and not args.no_secondary and args.workload in ("motion720", "motion4k", "dpd3"):
            # the same actor inside its on-device network (device channels)
            res["network"] = (motion_network if kind == "motion" else dpd_network)(p, args.steps, args.warmup)
        if world == 1 and kind == "motion" and not args.no_secondary:
            # BASELINE's metric also names DPD Msamples/s: the DPD configs
            # (configs[0], [2], [4] per GPU) measured the same way, compactly.
            sec = {}
            sub = argparse.Namespace(**vars(args))
            sub.steps, sub.warmup = 20, 3  # 20 back-to-back steps (a DPD-1 step is ~10 us)
            for name in ("dpd1", "dpd3", "dpd5"):
                sub.workload = name
                r = bench_dpd_ours(sub, WORKLOADS[name][1], rank, world, local)
                cb = cpu_dpd(WORKLOADS[name][1], 2, 1) if not args.no_cpu_baseline else None
                sec[name] = {"workload": WORKLOADS[name][1]["label"], "value": r["value"], "unit": r["unit"],
                             "ms_per_step": r["ms_per_step"], "e2e": r["e2e"]["value"],
                             "roofline": {k: r["roofline"][k] for k in ("bound", "achieved", "peak", "unit", "frac",
                                                                        "hbm_frac", "traffic")},
                             "cpu_baseline": cb}
                if name == "dpd3":
                    sec[name]["network"] = dpd_network(WORKLOADS[name][1], 5, 3)
            sec["resident_networks"] = resident_networks()
            res["secondary"] = sec
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
