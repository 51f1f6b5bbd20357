"""GPU: the C++ GPU-actor runtime (static schedule, per-actor streams,
event-encoded channel protocol, device-resident token counts) runs the
reference's two networks from host buffers and matches the oracle."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1611_03226_b200 import host_api as H

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("period,batch,blocks", [(256, 1, 8), (256, 4, 16), (4096, 8, 64), (64, 3, 21), (4, 5, 40)])
def test_dpd_network_equals_oracle(gpu, period, batch, blocks):
    x = O.synth_samples(period * blocks, 43)
    taps = O.random_taps(41)
    sched = O.random_schedule(5, 42)
    sched[1] = 1  # a single-branch block (extension; the oracle accepts it)
    got, ms, firings = H.dpd_run(x, taps, sched, period, batch, allow_single_branch=True)
    assert firings == blocks // batch
    np.testing.assert_array_equal(bits(got), bits(O.dpd(x, taps, sched, period)))


def test_dpd_network_t32(gpu):
    x = O.synth_samples(1024 * 16, 5)
    taps = O.random_taps(7, 32)
    got, _, _ = H.dpd_run(x, taps, [0x3FF], 1024, 4)
    np.testing.assert_array_equal(bits(got), bits(O.dpd(x, taps, [0x3FF], 1024)))


def test_dpd_network_rejects_bad_schedule(gpu):
    x = O.synth_samples(256, 1)
    with pytest.raises(H.HostRunError, match="invalid_argument"):
        H.dpd_run(x, O.random_taps(1), [0x7FF], 64)  # branch 11 (check_config)
    with pytest.raises(H.HostRunError, match="invalid_argument"):
        H.dpd_run(x, O.random_taps(1), [3], 48)  # samples not a multiple of period
    # k = 1 is outside the reference's [2,10] unless explicitly allowed
    with pytest.raises(H.HostRunError, match=r"outside \[2,10\]"):
        H.dpd_run(x, O.random_taps(1), [0x1], 64)
    got, _, _ = H.dpd_run(x, O.random_taps(1), [0x1], 64, allow_single_branch=True)
    np.testing.assert_array_equal(bits(got), bits(O.dpd(x, O.random_taps(1), [0x1], 64)))


@pytest.mark.parametrize("rate", [1, 4, 7])
@pytest.mark.parametrize("fmt", [1, 3])
def test_motion_network_equals_oracle(gpu, rate, fmt):
    w, h, n = 64, 48, 28
    f = O.synth_bytes(n * w * h * fmt, 2024)
    got, ms, delay_written = H.motion_run(f, w, h, fmt, 32, rate)
    want = O.motion_rgb(f, w, h) if fmt == 3 else O.motion_gray(f, w, h)
    np.testing.assert_array_equal(got, want)
    assert delay_written == n // rate  # one delay token per firing through the self-loop


@pytest.mark.parametrize("w,h,fmt,rate", [(640, 200, 3, 3), (1280, 136, 1, 5)])
def test_motion_network_large_frames(gpu, w, h, fmt, rate):
    # Frames with interior bands and several tiles: the TMA/TMEM kernel in
    # channel mode (region and delay token resolved from device phases).
    n = 4 * rate
    f = O.synth_bytes(n * w * h * fmt, w + h + rate)
    got, _, delay_written = H.motion_run(f, w, h, fmt, 32, rate)
    want = O.motion_rgb(f, w, h) if fmt == 3 else O.motion_gray(f, w, h)
    np.testing.assert_array_equal(got, want)
    assert delay_written == n // rate


def test_motion_acceptance6_through_runtime(gpu, hashes):
    import hashlib
    h = hashes["motion_acceptance6"]
    f = O.synth_bytes(h["frames"] * h["w"] * h["h"], h["seed"])
    for rate in (1, 4):
        got, _, _ = H.motion_run(f, h["w"], h["h"], 1, h["thr"], rate)
        assert hashlib.sha256(got.tobytes()).hexdigest() == h["out_sha256"]


@pytest.mark.parametrize("w,h,rate", [(64, 48, 1), (320, 120, 3), (96, 40, 2)])
def test_mixed_cpu_gpu_network(gpu, w, h, rate):
    # CPU actors (gray, census) and the GPU motion actor on shared device
    # channels: byte-exact masks, census counts from the CPU actor.
    n = 4 * rate
    rgb = O.synth_bytes(n * w * h * 3, 31 + w)
    got, counts, _ = H.motion_run_mixed(rgb, w, h, 32, rate)
    want = O.motion_rgb(rgb, w, h)
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(counts, (want.reshape(n, -1) != 0).sum(1))


def test_mixed_network_cpu_actor_fault(gpu):
    # fire throwing at firing 3 ends the run in ActorFault naming the actor
    # (proj/tests/test_runtime.cpp:251-277).
    w, h = 64, 48
    rgb = O.synth_bytes(8 * w * h * 3, 3)
    with pytest.raises(H.HostRunError, match="ActorFault: actor 'census' faulted: census: injected fault"):
        H.motion_run_mixed(rgb, w, h, 32, 1, fail_at_firing=3)


@pytest.mark.parametrize("rate", [1, 2, 3])
@pytest.mark.parametrize("sink_first", [False, True])
def test_delay_channel_orders_firings(gpu, rate, sink_first):
    """A delay channel of rate r > 1 orders producer firing i before consumer
    firing i (it needs r-1 of its tokens); only a rate-1 delay shifts by a
    whole firing.  Declaring the sink first must not change the stream."""
    firings = 7
    got = H.delay_chain_run(rate, sink_first, firings)
    want = np.concatenate([[np.uint64(2**64 - 1)], np.arange(1, firings * rate, dtype=np.uint64)])
    np.testing.assert_array_equal(got, want)


def _dynamic_cpu_expected(masks, rate, firings):
    # split -> branch b (x*(b+1) + running state, frozen while gated off) -> adder, int32 wrapping
    state = [0, 0]
    out = np.zeros(firings * rate, np.uint32)
    for i in range(firings):
        m = masks[i % len(masks)]
        x = (np.arange(rate, dtype=np.uint64) + i * rate + 1).astype(np.uint32)
        acc = np.zeros(rate, np.uint32)
        for b in (1, 2):
            if (m >> (b - 1)) & 1:
                state[b - 1] = (state[b - 1] + int(x.astype(np.uint64).sum())) & 0xFFFFFFFF
                acc += x * np.uint32(b + 1) + np.uint32(state[b - 1])
        out[i * rate:(i + 1) * rate] = acc
    return out.view(np.int32)


@pytest.mark.parametrize("rate", [1, 3])
def test_dynamic_cpu_actors_gated_ports_and_frozen_state(gpu, rate):
    # Dynamic-rate CPU actors (control read on the host, 0-or-r per port): the
    # reference's dynamic split / branch / adder shape with matched gating,
    # branches gated off for stretches (their state must stay frozen), and a
    # mask with no branch active (the adder still produces).
    from paper_1611_03226_b200 import host_api as H
    masks = [3, 1, 1, 0, 2, 3, 2, 2, 1]
    firings = 23
    got = H.dynamic_cpu_run(masks, rate, firings)
    np.testing.assert_array_equal(got, _dynamic_cpu_expected(masks, rate, firings))


def test_dynamic_cpu_actor_illegal_rate_is_actor_fault(gpu):
    from paper_1611_03226_b200 import host_api as H
    with pytest.raises(H.HostRunError) as e:
        H.dynamic_cpu_run([3, 1, 9], 2, 6)
    assert "ActorFault" in str(e.value) and "control" in str(e.value)


def test_bulk_kernel_adapter_cpu_actor(gpu):
    # df::bulk_kernel_adapter (proj/include/dynflow/runtime.hpp:97-108): whole
    # r-token regions to a batch kernel; a wrong output size faults the actor.
    from paper_1611_03226_b200 import host_api as H
    np.testing.assert_array_equal(H.bulk_kernel_run(5, 7), 2 * np.arange(35, dtype=np.int32))
    with pytest.raises(H.HostRunError) as e:
        H.bulk_kernel_run(5, 3, bad=True)
    assert "ActorFault" in str(e.value) and "doubler" in str(e.value) and "region is 20" in str(e.value)
