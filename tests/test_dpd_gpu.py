"""GPU parity: the sm_100a DPD actor vs the oracle (bit-exact float32,
which implies the reference's compare_samples 1e-5 criterion) and vs the
reference's own fixtures/hashes.  Pins follow proj/tests/test_dpd.cpp and
proj/tests/acceptance.cpp [8]-[10]."""
import hashlib

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5  # north_star / proj/src/bench.cpp:307-326 (we also require bit-exactness)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_parity(got, want):
    idx, worst = O.compare_samples(got, want, TOL)
    assert idx < 0, f"compare_samples FAIL at sample {idx}, worst rel err {worst}"
    bad = np.nonzero(bits(got) != bits(want))[0]
    assert bad.size == 0, f"{bad.size} float words differ, first at {bad[:5]}"


def run_gpu(x, taps, sched, period, chunk_blocks=0):
    from paper_1611_03226_b200 import dpd
    a = dpd.DpdActor(period, taps)
    out = np.empty_like(x)
    a.run_host(np.ascontiguousarray(x, np.float32), out, sched, chunk_blocks=chunk_blocks)
    a.check()
    return out


def test_acceptance8_bit_exact(gpu, hashes):
    h = hashes["dpd_acceptance8"]
    x = O.synth_samples(h["samples"], h["input_seed"])
    y = run_gpu(x, O.random_taps(h["taps_seed"]), O.random_schedule(*h["sched"]), h["period"])
    assert hashlib.sha256(y.tobytes()).hexdigest() == h["out_sha256"]


def test_period4096_random_schedule_hash(gpu, hashes):
    h = hashes["dpd_p4096_random"]
    x = O.synth_samples(h["samples"], h["input_seed"])
    y = run_gpu(x, O.random_taps(h["taps_seed"]), O.random_schedule(*h["sched"]), h["period"])
    assert hashlib.sha256(y.tobytes()).hexdigest() == h["out_sha256"]


@pytest.mark.parametrize("name", ["net_p256_s41", "gating_p64", "short_p4", "counts_p16"])
def test_reference_fixtures(gpu, small, name):
    period = int(small[f"dpd_{name}_period"][0])
    got = run_gpu(small[f"dpd_{name}_in"], small[f"dpd_{name}_taps"], small[f"dpd_{name}_sched"], period)
    assert_parity(got, small[f"dpd_{name}_out"])


@pytest.mark.parametrize("k", [1, 2, 10])
def test_single_branch_and_all_on(gpu, small, k):
    got = run_gpu(small["dpd_k_in"], small["dpd_k_taps"], [(1 << k) - 1], 64)
    assert_parity(got, small[f"dpd_k{k}_out"])


def ramp(blocks):
    return np.array([(1 << (1 + i % 10)) - 1 for i in range(blocks)], np.uint16)


@pytest.mark.parametrize("T", [10, 32, 1, 2, 7, 9, 31])
@pytest.mark.parametrize("period", [4096, 1000, 64, 8, 3])
def test_taps_and_periods_vs_oracle(gpu, T, period):
    blocks = max(4, 8192 // period)
    x = O.synth_samples(period * blocks, 1000 + T + period)
    taps = O.random_taps(77 + T, T)
    rng = np.random.default_rng(T * 1000 + period)
    sched = rng.integers(0, 1024, size=7).astype(np.uint16)  # includes k = 0, 1 and sparse masks
    assert_parity(run_gpu(x, taps, sched, period), O.dpd(x, taps, sched, period))


def test_ramp_schedule_1_to_10(gpu):
    period, blocks = 4096, 64
    x = O.synth_samples(period * blocks, 5)
    taps = O.random_taps(6)
    sched = ramp(blocks)
    assert_parity(run_gpu(x, taps, sched, period), O.dpd(x, taps, sched, period))


def test_chunked_firings_equal_one_batch(gpu):
    # FIR state carried across firings (proj/tests/test_dpd.cpp:140-177).
    period, blocks = 256, 37
    x = O.synth_samples(period * blocks, 11)
    taps = O.random_taps(12)
    sched = O.random_schedule(5, 13)
    want = O.dpd(x, taps, sched, period)
    for chunk in (1, 2, 5, 36):
        assert_parity(run_gpu(x, taps, sched, period, chunk_blocks=chunk), want)


@pytest.mark.parametrize("T", [10, 32])
@pytest.mark.parametrize("chunk", [0, 7, 64])
def test_long_gated_off_stretches(gpu, T, chunk):
    """Branches gated off for 32..150 blocks, inactive in whole firing
    batches, and never active: the frozen history must come from the last
    active block far back (several 32-token ballot steps of the in-kernel
    scan), from the carried FirState across batches, or stay zero
    (proj/src/dpd.cpp:264-279)."""
    period, blocks = 64, 200
    sched = np.full(blocks, 0x001, np.uint16)  # branch 1 always on
    sched[[0, 150, 151]] |= 1 << 4             # branch 5: gap of 149 blocks
    sched[[3, 35, 67, 199]] |= 1 << 6          # branch 7: gaps of exactly 32
    sched[[40, 41, 42]] |= 1 << 8              # branch 9: active once, gated after
    # branch 10 never active; branch 2 active only in the last block
    sched[199] |= 1 << 1
    x = O.synth_samples(period * blocks, 2024 + T)
    taps = O.random_taps(90 + T, T)
    assert_parity(run_gpu(x, taps, sched, period, chunk_blocks=chunk), O.dpd(x, taps, sched, period))


def _branch_tails(x, sched, period, first_block, T):
    """Per branch: the last T-1 raw samples of its active stream before
    `first_block` (None if it has fewer than T-1 -- then part of the state
    would come from zeros, which set_history cannot express; not used)."""
    xs = x.reshape(-1, period, 2)
    tails = []
    for b in range(1, 11):
        act = [p for p in range(first_block) if (int(sched[p % len(sched)]) >> (b - 1)) & 1]
        stream = xs[act].reshape(-1, 2) if act else np.zeros((0, 2), np.float32)
        tails.append(np.ascontiguousarray(stream[-(T - 1):]) if len(stream) >= T - 1 else None)
    return tails


@pytest.mark.parametrize("T,period", [(10, 256), (10, 64), (32, 256), (10, 4)])
def test_fire_halo_shard_equals_full_run(gpu, T, period):
    """df_dpd_fire_halo on a block-range shard, with per-branch halo tails of
    the stream before it, equals the shard of the full run (fast path: T=10
    with blocks >= T-1; prep path: T=32 and 4-sample blocks)."""
    from paper_1611_03226_b200 import device, dpd
    blocks = 40
    x = O.synth_samples(period * blocks, 77 + T + period)
    taps = O.random_taps(78, T)
    sched = np.array([0x3FF, 0x001, 0x2A5, 0x0F0, 0x100, 0x3FF, 0x003, 0x200, 0x3FF], np.uint16)
    want = O.dpd(x, taps, sched, period)
    b0 = 23
    tails = _branch_tails(x, sched, period, b0, T)
    bufs = [device.Buffer.from_array(t) if t is not None else None for t in tails]
    a = dpd.DpdActor(period, taps)
    nb = blocks - b0
    ctrl = device.Buffer(4 * nb)
    dpd.config_tokens(sched, b0, nb, ctrl)
    inp = device.Buffer.from_array(x[2 * period * b0:])
    out = device.Buffer(8 * period * nb)
    half = nb // 2  # two firings: the second continues from the state the first left
    a.fire_halo([bb.ptr.value if bb is not None else None for bb in bufs], ctrl, inp, out, half)
    a.fire(ctrl, inp, out, nb - half, ctrl_offset=4 * half, in_offset=8 * period * half,
           out_offset=8 * period * half)
    a.check()
    assert_parity(out.download(np.float32), want[2 * period * b0:])


@pytest.mark.parametrize("halo", [False, True])
def test_batch_over_65535_blocks(gpu, halo):
    """A firing of 70000 blocks is split into grid-sized sub-launches (grid.y
    <= 65535); each continues from the FirState the previous one advanced
    (and only the first takes the halo tails)."""
    from paper_1611_03226_b200 import device, dpd
    period, blocks, T = 16, 70000, 10
    x = O.synth_samples(period * blocks, 4711)
    taps = O.random_taps(4712, T)
    rng = np.random.default_rng(4713)
    sched = rng.integers(0, 1024, size=97).astype(np.uint16)
    sched[60:] &= 0x1FF  # branch 10 gated off in a long stretch of every cycle
    if not halo:
        assert_parity(run_gpu(x, taps, sched, period), O.dpd(x, taps, sched, period))
        return
    b0 = 5
    tails = _branch_tails(x, sched, period, b0, T)
    bufs = [device.Buffer.from_array(t) if t is not None else None for t in tails]
    a = dpd.DpdActor(period, taps)
    nb = blocks - b0
    ctrl = device.Buffer(4 * nb)
    dpd.config_tokens(sched, b0, nb, ctrl)
    inp = device.Buffer.from_array(x[2 * period * b0:])
    out = device.Buffer(8 * period * nb)
    a.fire_halo([bb.ptr.value if bb is not None else None for bb in bufs], ctrl, inp, out, nb)
    a.check()
    want = O.dpd(x, taps, sched, period)
    assert_parity(out.download(np.float32), want[2 * period * b0:])


def test_run_host_schedule_change_between_runs(gpu):
    """df_dpd_run_host reuses the control tokens of an identical schedule and
    regenerates them when the schedule (same length) or the block count
    changes."""
    from paper_1611_03226_b200 import dpd
    period, T = 256, 10
    taps = O.random_taps(55, T)
    a = dpd.DpdActor(period, taps)
    sa = np.array([0x3FF, 0x001, 0x0F0], np.uint16)
    sb = np.array([0x002, 0x300, 0x155], np.uint16)
    for sched, blocks in ((sa, 12), (sb, 12), (sa, 12), (sa, 7), (sb, 7)):
        x = O.synth_samples(period * blocks, int(sched[0]) + blocks)
        a.reset()
        out = np.empty_like(x)
        a.run_host(x, out, sched)
        a.check()
        assert_parity(out, O.dpd(x, taps, sched, period))


@pytest.mark.parametrize("splits", [(5,), (5, 4), (1, 1, 7), (3, 3, 3)])
def test_run_host_split_stream_equals_one_run(gpu, splits):
    """Several df_dpd_run_host calls without a reset continue the FIR
    history AND the schedule position, so a stream split at any block count
    (not only at multiples of the schedule length) equals one oracle run."""
    from paper_1611_03226_b200 import dpd
    period, T = 128, 10
    taps = O.random_taps(77, T)
    sched = np.array([0x3FF, 0x001, 0x0F0, 0x206], np.uint16)  # length 4
    blocks = sum(splits) + 2
    x = O.synth_samples(period * blocks, 78)
    want = O.dpd(x, taps, sched, period)
    a = dpd.DpdActor(period, taps)
    got = np.empty_like(x)
    b0 = 0
    for nb in list(splits) + [2]:
        lo, hi = 2 * period * b0, 2 * period * (b0 + nb)
        out = np.empty(hi - lo, np.float32)
        a.run_host(np.ascontiguousarray(x[lo:hi]), out, sched)
        got[lo:hi] = out
        b0 += nb
    a.check()
    assert_parity(got, want)


def test_gating_invariance_acceptance9(gpu):
    # proj/tests/acceptance.cpp:398-450: branch 7 toggled; inactive periods
    # must be bit-identical when its taps change.
    period, branch = 4096, 7
    sched = []
    for p in range(8):
        t = int(O.random_schedule(8, 900 + p)[0])
        if p % 2 == 0:
            t |= 1 << (branch - 1)
        else:
            t &= ~(1 << (branch - 1))
            if bin(t).count("1") < 2:
                t |= 0b11
        sched.append(t)
    x = O.synth_samples(period * 8, 902)
    taps = O.random_taps(901)
    base = run_gpu(x, taps, sched, period)
    alt = taps.copy()
    alt[branch - 1] = O.random_taps(903)[0]
    changed = run_gpu(x, alt, sched, period)
    for p in range(8):
        seg = slice(2 * p * period, 2 * (p + 1) * period)
        differs = not np.array_equal(bits(base[seg]), bits(changed[seg]))
        assert differs == bool(sched[p] >> (branch - 1) & 1), p


def test_zero_and_impulse(gpu):
    # proj/tests/test_dpd.cpp:299-331
    taps = O.random_taps(11)
    x = np.zeros(2 * 128, np.float32)
    assert not run_gpu(x, taps, [0x3FF], 64).any()
    x[0] = 1.0
    y = run_gpu(x, taps, [0x3FF], 64).reshape(-1, 2)
    want = np.zeros((64, 2), np.float64)
    want[:10] = taps.astype(np.float64).sum(0)
    idx, worst = O.compare_samples(y[:64].astype(np.float32), want.astype(np.float32), TOL)
    assert idx < 0, worst


def test_control_token_beyond_branch_10_is_control_error(gpu):
    from paper_1611_03226_b200 import ControlError, dpd
    a = dpd.DpdActor(64, O.random_taps(1))
    x = O.synth_samples(128, 1)
    out = np.empty_like(x)
    a.run_host(x, out, [0x7FF])
    with pytest.raises(ControlError):
        a.check()


def test_raw_fire_and_config_actor_on_device(gpu):
    from paper_1611_03226_b200 import dpd
    from paper_1611_03226_b200.device import Buffer, Stream
    period, blocks = 512, 20
    x = O.synth_samples(period * blocks, 3)
    taps = O.random_taps(4)
    sched = O.random_schedule(6, 5)
    s = Stream()
    a = dpd.DpdActor(period, taps)
    xin = Buffer.from_array(x, stream=s)
    out = Buffer(x.nbytes)
    ctrl = Buffer(4 * blocks)
    dpd.config_tokens(sched, 0, blocks, ctrl, stream=s)
    a.fire(ctrl, xin, out, 7, s)
    a.fire(ctrl, xin, out, blocks - 7, s, ctrl_offset=4 * 7, in_offset=8 * period * 7, out_offset=8 * period * 7)
    s.synchronize()
    assert_parity(out.download(np.float32), O.dpd(x, taps, sched, period))
    st = a.state()
    assert st.shape == (10, 9, 2)


@pytest.mark.parametrize("T,period", [(10, 256), (32, 1000), (10, 5)])
def test_channel_bound_firing(gpu, T, period):
    """Batched firing over device channels: control tokens and block tokens
    are consumed, and regions resolved, on the device."""
    from paper_1611_03226_b200 import dpd
    from paper_1611_03226_b200.channel import DeviceChannel
    from paper_1611_03226_b200.device import Stream
    import ctypes as C
    from paper_1611_03226_b200._lib import call
    K, rounds = 6, 5
    x = O.synth_samples(period * K * rounds, 21)
    taps = O.random_taps(22, T)
    sched = list(O.random_schedule(4, 23)) + [1, 0x200, 0]  # incl. k = 1 and empty masks
    s = Stream()
    ctrl = DeviceChannel(4, K)
    cin = DeviceChannel(8 * period, K)
    cout = DeviceChannel(8 * period, K)
    a = dpd.DpdActor(period, taps)
    got = np.empty_like(x)
    for r in range(rounds):
        w = ctrl.write_start(K)
        toks = np.array([sched[(r * K + i) % len(sched)] for i in range(K)], np.uint32)
        call("df_memcpy_h2d", C.c_void_p(w.dptr), toks.ctypes.data_as(C.c_void_p), toks.nbytes, s.handle)
        ctrl.write_end(w, s)
        w = cin.write_start(K)
        blk = np.ascontiguousarray(x[2 * r * K * period: 2 * (r + 1) * K * period])
        call("df_memcpy_h2d", C.c_void_p(w.dptr), blk.ctypes.data_as(C.c_void_p), blk.nbytes, s.handle)
        cin.write_end(w, s)
        a.fire_channels(ctrl, cin, cout, K, s)
        rd = cout.read_start(K)
        part = np.empty(2 * K * period, np.float32)
        call("df_memcpy_d2h", part.ctypes.data_as(C.c_void_p), C.c_void_p(rd.dptr), part.nbytes, s.handle)
        cout.read_end(rd, s)
        s.synchronize()
        got[2 * r * K * period: 2 * (r + 1) * K * period] = part
    for ch in (ctrl, cin, cout):
        ch.check()
        st = ch.stats()
        assert st.tokens_written == K * rounds and st.tokens_read == K * rounds and st.tokens_available == 0
    a.check()
    assert_parity(got, O.dpd(x, taps, sched, period))


def test_block_shard_with_history_halo(gpu):
    """A block-range shard primed from the T-1 raw samples before it
    (df_dpd_set_history) equals the matching slice of the full run; for a
    dynamic schedule each branch takes the tail of its last active block."""
    from paper_1611_03226_b200 import dpd, shard
    from paper_1611_03226_b200.device import Buffer
    for T, sched in [(32, [0x3FF]), (10, list(O.random_schedule(7, 3)) + [1])]:
        period, blocks, s_block = 128, 16, 9
        x = O.synth_samples(period * blocks, 8)
        taps = O.random_taps(9, T)
        full = O.dpd(x, taps, sched, period)
        a = dpd.DpdActor(period, taps)
        xb = Buffer.from_array(x)
        for b in range(1, 11):
            hb = shard.dpd_halo_block(sched, s_block, b)
            if hb is not None:
                a.set_history(xb, period, 1 << (b - 1), offset=8 * period * hb)
        rest = blocks - s_block
        ctrl = Buffer.from_array(np.array([sched[(s_block + i) % len(sched)] for i in range(rest)], np.uint32))
        out = Buffer(8 * period * rest)
        a.fire(ctrl, xb, out, rest, in_offset=8 * period * s_block)
        got = out.download(np.float32)
        assert_parity(got, full[2 * period * s_block:])


@pytest.mark.parametrize("T", [10, 32])
def test_grid_orders_agree(gpu, T):
    """Short firings (<= 4096 CTAs) run block-major with a next-wave L2
    prefetch, long ones tile-major: the same stream fired as one 8192-CTA
    batch and in 64-block chunks must be bit-identical, and match the oracle
    (a ramp plus gated-off stretches exercises the FirState hand-off)."""
    period, blocks = 4096, 2048  # 4 tiles per block: 8192 CTAs in one batch
    x = O.synth_samples(period * blocks, 2100 + T)
    taps = O.random_taps(2200 + T, T)
    sched = np.array([(1 << (1 + i % 10)) - 1 for i in range(10)] + [1, 0x200, 0x3FF, 2], np.uint16)
    whole = run_gpu(x, taps, sched, period, chunk_blocks=blocks)
    chunked = run_gpu(x, taps, sched, period, chunk_blocks=64)
    assert np.array_equal(bits(whole), bits(chunked))
    n = 96 * period
    assert_parity(whole[:2 * n], O.dpd(x[:2 * n], taps, sched, period))


def test_kernel_name_follows_grid(gpu):
    """df_dpd_kernel_name names the main kernel of the last firing: the
    one-wave kernel for a DPD-1-sized batch (2^20 samples, period 4096),
    the tiled main kernel for a batch over one wave, the generic kernel
    for tap counts other than 10/32 -- and each output stays bit-exact."""
    from paper_1611_03226_b200 import dpd
    taps = O.random_taps(2300, 10)
    sched = np.array([3], np.uint16)
    a = dpd.DpdActor(4096, taps)
    assert a.kernel_name == ""
    for blocks, want in ((256, "dpd_wave_kernel"), (4096, "dpd_main_kernel")):
        x = O.synth_samples(4096 * blocks, 2400 + blocks)
        out = np.empty_like(x)
        a.reset()
        a.run_host(np.ascontiguousarray(x, np.float32), out, sched, chunk_blocks=blocks)
        a.check()
        assert a.kernel_name == want
        n = 8 * 4096
        assert_parity(out[:2 * n], O.dpd(x[:2 * n], taps, sched, 4096))
    g = dpd.DpdActor(64, O.random_taps(2301, 7))
    x = O.synth_samples(64 * 16, 2500)
    out = np.empty_like(x)
    g.run_host(np.ascontiguousarray(x, np.float32), out, sched)
    assert g.kernel_name == "dpd_main_generic_kernel"


def test_empty_firings_keep_the_fir_state(gpu):
    """Zero samples / zero blocks fire nothing: the FIR history, the
    run_host schedule position and the output of the next firing are
    unchanged (oracle over the whole stream)."""
    from paper_1611_03226_b200 import dpd
    from paper_1611_03226_b200.device import Buffer
    period, blocks = 64, 12
    x = O.synth_samples(period * blocks, 2600)
    taps = O.random_taps(2601)
    sched = np.array([3, 0x3FF, 0x101, 6, 0x200], np.uint16)
    want = O.dpd(x, taps, sched, period)
    a = dpd.DpdActor(period, taps)
    got = np.empty_like(x)
    h = 2 * period * 5
    a.run_host(np.ascontiguousarray(x[:h]), got[:h], sched)
    a.run_host(np.empty(0, np.float32), np.empty(0, np.float32), sched)
    scratch = Buffer(64)
    a.fire(scratch, scratch, scratch, 0)
    a.run_host(np.ascontiguousarray(x[h:]), got[h:], sched)
    a.check()
    assert_parity(got, want)
