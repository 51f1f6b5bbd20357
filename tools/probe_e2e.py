"""Probe: df_dpd_run_host time vs chunk size, and raw pinned H2D/D2H copy
times for the same bytes (where the DPD-1 e2e time goes)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1611_03226_b200 import device, dpd

N, period = 1 << 20, 65536
actor = dpd.DpdActor(period, np.random.default_rng(808).uniform(-0.5, 0.5, (10, 10, 2)).astype(np.float32))
hin = device.PinnedArray(2 * N, np.float32)
hout = device.PinnedArray(2 * N, np.float32)
hin.array[:] = np.random.default_rng(0).uniform(-1, 1, 2 * N).astype(np.float32)
sched = np.array([3], np.uint16)


def t(fn, reps=20):
    fn()
    ts = []
    for _ in range(reps):
        a = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - a)
    return statistics.median(ts) * 1e6


for cb in (0, 16, 8, 4, 2, 1):
    us = t(lambda: actor.run_host(hin.array, hout.array, sched, chunk_blocks=cb))
    print(f"run_host chunk_blocks={cb}: {us:.1f} us  -> {N / us:.0f} Msps")
d_in = torch.empty(2 * N, dtype=torch.float32, device="cuda")
th = torch.from_numpy(hin.array)
to = torch.from_numpy(hout.array)
print(f"H2D 8MB: {t(lambda: (d_in.copy_(th, non_blocking=True), torch.cuda.synchronize())):.1f} us")
print(f"D2H 8MB: {t(lambda: (to.copy_(d_in, non_blocking=True), torch.cuda.synchronize())):.1f} us")
s2 = torch.cuda.Stream()
d_out = torch.empty_like(d_in)


def both():
    with torch.cuda.stream(s2):
        to.copy_(d_out, non_blocking=True)
    d_in.copy_(th, non_blocking=True)
    torch.cuda.synchronize()


print(f"H2D+D2H concurrent 8MB each: {t(both):.1f} us")
print(f"empty sync: {t(lambda: torch.cuda.synchronize()):.1f} us")


# The same 3-stream pipeline with torch streams (copy kernel as the "fire").
def pipe(nch, slots=3):
    h2d, cs, d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    n = 2 * N // nch
    din = [torch.empty(n, device="cuda") for _ in range(slots)]
    dout = [torch.empty(n, device="cuda") for _ in range(slots)]
    ev_in = [torch.cuda.Event() for _ in range(nch)]
    ev_c = [torch.cuda.Event() for _ in range(nch)]
    ev_o = [torch.cuda.Event() for _ in range(nch)]

    def run():
        for c in range(nch):
            i = c % slots
            with torch.cuda.stream(h2d):
                if c >= slots:
                    h2d.wait_event(ev_c[c - slots])
                din[i].copy_(th[c * n:(c + 1) * n], non_blocking=True)
                ev_in[c].record(h2d)
            with torch.cuda.stream(cs):
                cs.wait_event(ev_in[c])
                if c >= slots:
                    cs.wait_event(ev_o[c - slots])
                dout[i].copy_(din[i])
                ev_c[c].record(cs)
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_c[c])
                to[c * n:(c + 1) * n].copy_(dout[i], non_blocking=True)
                ev_o[c].record(d2h)
        torch.cuda.synchronize()

    return t(run)


for nch in (1, 2, 4, 8, 16):
    print(f"torch 3-stream pipeline, {nch} chunks: {pipe(nch):.1f} us")


# Round-robin: chunk c on stream c % ns with its own slot; no events.
def rr(nch, ns):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    n = 2 * N // nch
    din = [torch.empty(n, device="cuda") for _ in range(ns)]
    dout = [torch.empty(n, device="cuda") for _ in range(ns)]

    def run():
        for c in range(nch):
            i = c % ns
            with torch.cuda.stream(ss[i]):
                din[i].copy_(th[c * n:(c + 1) * n], non_blocking=True)
                dout[i].copy_(din[i])
                to[c * n:(c + 1) * n].copy_(dout[i], non_blocking=True)
        torch.cuda.synchronize()

    return t(run)


for ns in (2, 3, 4):
    for nch in (2, 4, 8, 16):
        if nch >= ns:
            print(f"torch round-robin {ns} streams, {nch} chunks: {rr(nch, ns):.1f} us")
s3 = device.Stream() if hasattr(device, "Stream") else None
for cb in (8, 4, 2):
    us = t(lambda: actor.run_host(hin.array, hout.array, sched, chunk_blocks=cb, stream=s3))
    print(f"run_host on a created stream, chunk_blocks={cb}: {us:.1f} us")
