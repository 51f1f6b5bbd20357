"""GPU: device-resident networks (csrc/netrt.cu) -- persistent actors with
device-side control dispatch, blocking channels, end of stream, drain,
abort and fault propagation.

Pins follow the reference's own tests:
  * the reference's 15-actor / 56-channel DPD network == oracle_dpd
    (proj/tests/test_dpd.cpp:390-408, acceptance.cpp [8] and [9]) and its
    control-token counts (test_dpd.cpp:427-455);
  * the 5-actor motion network with its delay channel == oracle
    (test_motion.cpp:194-217, acceptance.cpp [6] at r = 1 and 4);
  * channel KATs on device rings under concurrency and dynamic rates
    (test_channel.cpp:121-158, :209-259, :265-375; acceptance.cpp [3], [4]);
  * fault injection / ControlError / RunAborted (test_runtime.cpp:251-277,
    channel.cpp:170-177).
"""
import ctypes as C
import hashlib
import threading
import time

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ---------------------------------------------------------------- DPD network
@pytest.mark.parametrize("seed", [41, 42, 43])
def test_resident_dpd_network_equals_oracle(gpu, seed):
    from paper_1611_03226_b200 import host_api as H
    period, blocks = 256, 12
    x = O.synth_samples(period * blocks, seed + 1)
    taps = O.random_taps(seed)
    sched = O.random_schedule(5, seed + 2)  # k in [2, 10], the reference's check_config range
    got, ms, firings, tokens = H.dpd_run_resident(x, taps, sched, period)
    np.testing.assert_array_equal(bits(got), bits(O.dpd(x, taps, sched, period)))
    # Every actor fires once per block: dynamic actors consume one control
    # token per firing even when all their ports are at rate 0.
    assert all(v == blocks for v in firings.values()), firings
    # Channel tokens: split_bXX_{re,im} carry exactly the blocks where b is on.
    masks = np.array([sched[i % len(sched)] for i in range(blocks)])
    for b in range(1, 11):
        on = int(((masks >> (b - 1)) & 1).sum())
        assert tokens[2 + 2 * (b - 1)] == on and tokens[3 + 2 * (b - 1)] == on, b
        assert tokens[22 + 2 * (b - 1)] == on, b  # bXX_adder_re
    assert tokens[0] == blocks and tokens[42] == blocks  # src_split_re, adder_sink_re
    assert tokens[44:].tolist() == [blocks] * 12  # the 12 control channels
    assert ms > 0


def test_resident_dpd_acceptance8(gpu, hashes):
    from paper_1611_03226_b200 import host_api as H
    h = hashes["dpd_acceptance8"]
    x = O.synth_samples(h["samples"], h["input_seed"])
    y, _, _, _ = H.dpd_run_resident(x, O.random_taps(h["taps_seed"]), O.random_schedule(*h["sched"]), h["period"])
    assert hashlib.sha256(y.tobytes()).hexdigest() == h["out_sha256"]


def test_resident_dpd_gating_invariance_acceptance9(gpu):
    # acceptance.cpp:398-450: branch 7 toggled per period; inactive periods
    # are bit-identical when its taps change (its state stays frozen).
    from paper_1611_03226_b200 import host_api as H
    period, branch = 4096, 7
    sched = []
    for p in range(8):
        t = int(O.random_schedule(8, 900 + p)[0])
        t = t | (1 << (branch - 1)) if p % 2 == 0 else t & ~(1 << (branch - 1))
        if bin(t).count("1") < 2:
            t |= 0b11
        sched.append(t)
    x = O.synth_samples(period * 8, 902)
    taps = O.random_taps(901)
    base, _, _, _ = H.dpd_run_resident(x, taps, sched, period)
    np.testing.assert_array_equal(bits(base), bits(O.dpd(x, taps, sched, period)))
    alt = taps.copy()
    alt[branch - 1] = O.random_taps(903)[0]
    changed, _, _, _ = H.dpd_run_resident(x, alt, sched, period)
    for p in range(8):
        seg = slice(2 * p * period, 2 * (p + 1) * period)
        differs = not np.array_equal(bits(base[seg]), bits(changed[seg]))
        assert differs == bool(sched[p] >> (branch - 1) & 1), p


@pytest.mark.parametrize("T,period,ctas", [(32, 64, 3), (10, 4, 1), (10, 1000, 5)])
def test_resident_dpd_extensions_and_short_blocks(gpu, T, period, ctas):
    # T = 32 and k = 1 masks (extensions); blocks shorter than T-1 chain the
    # history through older state (dpd.cpp:108-120); uneven CTA splits.
    from paper_1611_03226_b200 import host_api as H
    blocks = 9
    x = O.synth_samples(period * blocks, 7 + T)
    taps = O.random_taps(5, T)
    sched = np.array([0x3FF, 0x001, 0x2A5, 0x200, 0x0F0, 0x001, 0x3FF, 0x155, 0x300], np.uint16)
    got, _, fir, _ = H.dpd_run_resident(x, taps, sched, period, allow_single_branch=True, branch_ctas=ctas)
    np.testing.assert_array_equal(bits(got), bits(O.dpd(x, taps, sched, period)))
    assert fir["branch10"] == blocks


def test_resident_dpd_rejects_single_branch_by_default(gpu):
    from paper_1611_03226_b200 import host_api as H
    x = O.synth_samples(64, 1)
    with pytest.raises(H.HostRunError, match=r"outside \[2,10\]"):
        H.dpd_run_resident(x, O.random_taps(1), [0x1], 64)


# ------------------------------------------------------------- motion network
def test_resident_motion_fixture_64x48(gpu, small):
    from paper_1611_03226_b200 import host_api as H
    got, ms, fir = H.motion_run_resident(small["motion_64x48_in"], 64, 48, ctas=4)
    np.testing.assert_array_equal(got, small["motion_64x48_out"].reshape(-1))
    assert fir == {"source": 16, "gauss": 16, "thres": 16, "med": 16, "sink": 16}


@pytest.mark.parametrize("w,h", [(40, 9), (8, 5), (37, 23), (1280, 72), (32, 5), (48, 5), (64, 7), (336, 41)])
def test_resident_motion_sizes_vs_oracle(gpu, w, h):
    # 16-px gauss/median actors (W % 16 == 0: 1280x72, 32x5 and 48x5 at the
    # row / column minimum, 64x7 with two chunks per row, 336x41), word-wise
    # (W % 4 == 0: 40x9, 8x5) and the byte-wise fallback (37x23).
    from paper_1611_03226_b200 import host_api as H
    f = O.synth_bytes(6 * w * h, 7000 + w)
    out, _, _ = H.motion_run_resident(f, w, h, 32, ctas=4)
    np.testing.assert_array_equal(out, O.motion_gray(f, w, h, 32))


@pytest.mark.parametrize("rate", [1, 4])
def test_resident_motion_acceptance6(gpu, hashes, rate):
    # acceptance.cpp:328-341 at r = 1 and 4: at r = 4 the thres actor's prev
    # region is [copied delay token, f0..f2] (the Fig. 2 walk, channel.cpp:26-32).
    from paper_1611_03226_b200 import host_api as H
    h = hashes["motion_acceptance6"]
    f = O.synth_bytes(h["frames"] * h["w"] * h["h"], h["seed"])
    out, _, fir = H.motion_run_resident(f, h["w"], h["h"], h["thr"], rate=rate)
    assert hashlib.sha256(out.tobytes()).hexdigest() == h["out_sha256"]
    assert fir["sink"] == h["frames"] // rate


# ------------------------------------------------- channel KATs on device rings
def _counters():
    from paper_1611_03226_b200 import device
    buf = device.Buffer(16)
    buf.zero()
    return buf


def _read(buf):
    return buf.download(np.uint64, 2)


@pytest.mark.parametrize("rate", [1, 4, 7])
@pytest.mark.parametrize("delay", [False, True])
def test_concurrent_producer_consumer_stream(gpu, rate, delay):
    """test_channel.cpp:322-375 on a device ring: producer and consumer are
    concurrent persistent actors with randomized stalls; the producer closes
    after its last batch, the consumer reads until end of stream."""
    from paper_1611_03226_b200 import netrt
    from paper_1611_03226_b200.channel import DeviceChannel
    token, batches, seed = 8, 3000, 42 + rate + (100 if delay else 0)
    ch = DeviceChannel(token, rate, delay)
    pc, cc = _counters(), _counters()
    net = netrt.Net()
    net.add(netrt.DF_ACT_TEST_PRODUCE, netrt.Test(seed, pc.at(0).value, 63, 0, 0), outputs=[ch], limit=batches)
    net.add(netrt.DF_ACT_TEST_CONSUME, netrt.Test(seed, cc.at(0).value, 63, int(delay), 0), inputs=[ch])
    net.run(timeout_s=20)
    produced, _ = _read(pc)
    consumed, bad = _read(cc)
    total = batches * rate + (1 if delay else 0)
    assert produced == batches * rate
    assert bad == 0
    assert consumed == (total // rate) * rate
    st = ch.stats()
    assert st.tokens_available == total - consumed  # residual below one batch
    assert st.closed == 1
    assert net.stats(0)[0] == batches and net.stats(1)[0] == total // rate


def _config(schedule):
    from paper_1611_03226_b200 import device
    s = np.ascontiguousarray(np.asarray(schedule, np.uint16))
    return device.Buffer.from_array(s)


@pytest.mark.parametrize("rate", [1, 3])
def test_dynamic_rates_gated_producer_static_consumer(gpu, rate):
    """A dynamic producer whose control token gates its output to 0 or r
    (control_dispatch on the device) feeding a STATIC consumer: the consumer
    fires only when r tokens exist, so the two fire different numbers of
    times -- general data-dependent rates, not lock step -- and it stops at
    end of stream once the producer closes."""
    from paper_1611_03226_b200 import netrt
    from paper_1611_03226_b200.channel import DeviceChannel
    rng = np.random.default_rng(5 + rate)
    sched = rng.integers(0, 2, 257).astype(np.uint16)
    firings = 600
    ctrl = DeviceChannel(4, 1)
    data = DeviceChannel(8, rate)
    sbuf = _config(sched)
    pc, cc = _counters(), _counters()
    net = netrt.Net()
    net.add(netrt.DF_ACT_DPD_CONFIG, netrt.Config(sbuf.at(0).value, sched.size), outputs=[ctrl], limit=firings)
    prod = net.add(netrt.DF_ACT_TEST_PRODUCE, netrt.Test(9, pc.at(0).value, 15, 0, 0), control=ctrl, outputs=[data])
    net.control_table(prod, [(0, 0, 1), (0, 1, 1)])  # token 0: output at rate 0; token 1: at rate r
    net.add(netrt.DF_ACT_TEST_CONSUME, netrt.Test(9, cc.at(0).value, 7, 0, 0), ctas=2, inputs=[data])
    net.run(timeout_s=20)
    on = int(np.array([sched[i % sched.size] for i in range(firings)]).sum())
    assert _read(pc)[0] == on * rate
    consumed, bad = _read(cc)
    assert bad == 0 and consumed == on * rate
    assert net.stats(prod)[0] == firings  # one firing per control token, gated or not
    assert net.stats(2)[0] == on


def test_control_token_outside_domain_faults_the_actor(gpu):
    """ControlError (model.cpp:240-265): a token with no legal rates faults
    the dynamic actor; every other actor is aborted instead of hanging."""
    from paper_1611_03226_b200 import ControlError, netrt
    from paper_1611_03226_b200.channel import DeviceChannel
    sched = np.array([1, 0, 1, 5, 1], np.uint16)  # 5 is outside the 2-entry domain
    ctrl, data = DeviceChannel(4, 1), DeviceChannel(8, 1)
    sbuf = _config(sched)
    pc, cc = _counters(), _counters()
    net = netrt.Net()
    net.add(netrt.DF_ACT_DPD_CONFIG, netrt.Config(sbuf.at(0).value, sched.size), outputs=[ctrl], limit=100)
    prod = net.add(netrt.DF_ACT_TEST_PRODUCE, netrt.Test(1, pc.at(0).value, 0, 0, 0), control=ctrl, outputs=[data])
    net.control_table(prod, [(0, 0, 1), (0, 1, 1)])
    net.add(netrt.DF_ACT_TEST_CONSUME, netrt.Test(1, cc.at(0).value, 0, 0, 0), inputs=[data])
    with pytest.raises(ControlError):
        net.run(timeout_s=10)
    actor, code, token = net.fault()
    assert (actor, code, token) == (prod, 5, 5)
    assert net.stats(prod)[0] == 3  # fired on tokens 1, 0, 1; faulted on 5


def test_host_abort_wakes_blocked_actors(gpu):
    """channel.cpp:170-177 / test_channel.cpp:238-246: abort wakes a blocked
    reader with RunAborted.  The producer holds 20 s before each firing; the
    consumer blocks in read_start until df_net_abort (from another thread)."""
    from paper_1611_03226_b200 import RunAborted, netrt
    from paper_1611_03226_b200.channel import DeviceChannel
    ch = DeviceChannel(8, 1)
    pc, cc = _counters(), _counters()
    net = netrt.Net()
    net.add(netrt.DF_ACT_TEST_PRODUCE, netrt.Test(3, pc.at(0).value, 0, 0, 20_000_000_000), outputs=[ch], limit=5)
    net.add(netrt.DF_ACT_TEST_CONSUME, netrt.Test(3, cc.at(0).value, 0, 0, 0), inputs=[ch])
    t = threading.Timer(0.3, net.abort)
    t.start()
    t0 = time.time()
    with pytest.raises(RunAborted):
        net.run(timeout_s=60)
    assert time.time() - t0 < 15
    assert _read(cc)[0] == 0


def test_watchdog_ends_a_deadlocked_network(gpu):
    """A cycle whose delay token cannot cover one firing (rate 2): the
    reference blocks forever (validate() now rejects it; the raw C ABI does
    not validate).  The device watchdog faults the waiting actor instead of
    hanging the GPU."""
    from paper_1611_03226_b200 import WatchdogTimeout, netrt
    from paper_1611_03226_b200.channel import DeviceChannel
    ch = DeviceChannel(8, 2, has_delay=True)  # one initial token, consumer needs 2
    cc = _counters()
    net = netrt.Net()
    net.add(netrt.DF_ACT_TEST_CONSUME, netrt.Test(3, cc.at(0).value, 0, 1, 0), inputs=[ch])
    t0 = time.time()
    with pytest.raises(WatchdogTimeout):
        net.run(timeout_s=0.3)
    assert time.time() - t0 < 10
    assert net.fault()[1] == 7


def test_end_of_stream_on_host_read_after_drain(gpu):
    """read_start on a closed, drained channel is end of stream (nullopt ->
    DF_EOS); with r tokens left it still succeeds (test_channel.cpp:377-388)."""
    from paper_1611_03226_b200 import EndOfStream, netrt
    from paper_1611_03226_b200.channel import DeviceChannel
    a = DeviceChannel(4, 2)  # producer -> consumer: drained by the consumer
    b = DeviceChannel(4, 2)  # producer2 -> (nobody): closed with tokens left
    pa, pb, ca = _counters(), _counters(), _counters()
    net = netrt.Net()
    net.add(netrt.DF_ACT_TEST_PRODUCE, netrt.Test(4, pa.at(0).value, 0, 0, 0), outputs=[a], limit=3)
    net.add(netrt.DF_ACT_TEST_CONSUME, netrt.Test(4, ca.at(0).value, 0, 0, 0), inputs=[a])
    net.add(netrt.DF_ACT_TEST_PRODUCE, netrt.Test(5, pb.at(0).value, 0, 0, 0), outputs=[b], limit=1)
    net.run(timeout_s=10)
    with pytest.raises(EndOfStream):
        a.read_start(2)
    r = b.read_start(2)  # two tokens remain after close
    b.read_end(r)
    with pytest.raises(EndOfStream):
        b.read_start(2)


def test_network_too_large_for_one_wave_is_rejected(gpu):
    from paper_1611_03226_b200 import InvalidArgument, netrt
    from paper_1611_03226_b200.channel import DeviceChannel
    ch = DeviceChannel(8, 1)
    pc, cc = _counters(), _counters()
    net = netrt.Net()
    net.add(netrt.DF_ACT_TEST_PRODUCE, netrt.Test(3, pc.at(0).value, 0, 0, 0), ctas=100000, outputs=[ch], limit=1)
    net.add(netrt.DF_ACT_TEST_CONSUME, netrt.Test(3, cc.at(0).value, 0, 0, 0), inputs=[ch])
    with pytest.raises(InvalidArgument, match="co-resident"):
        net.run()
