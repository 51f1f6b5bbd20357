"""CPU: the C++ host runtime's model rules (libdf_host.so), mirroring
proj/tests/test_model.cpp -- no device needed."""
import pytest

from paper_1611_03226_b200 import host_api as H


def test_gpu_dpd_network_shape_validates():
    assert H.validate_demo(0) == 0


def test_undelayed_cycle_and_static_control_port_are_violations():
    assert H.validate_demo(1) == 2


def test_delayed_self_loop_is_legal():
    assert H.validate_demo(2) == 0


def test_cycles_through_rate2_delay_channels_are_violations():
    # A delay token covers one firing only at rate 1: a cycle whose delay
    # channels all have rate > 1 blocks forever in the reference's read_start.
    assert H.validate_demo(5) == 1
    assert H.validate_demo(6) == 1


def test_batched_control_rate_needs_matching_port_rates():
    # The reference requires control rate 1 (model.cpp:133-134).  A device-
    # controlled GPU actor may batch r reference firings (r control tokens,
    # r tokens on every regular port); any other control rate is rejected.
    assert H.validate_demo(7) == 0
    assert H.validate_demo(8) == 1


def test_unknown_channel_is_build_error():
    assert H.validate_demo(3) == -1
    assert b"BuildError" in H.lib().dfh_last_error()


def test_validate_cpu_actor_rules():
    # A CPU actor marked device_control (a CPU actor reads its control token
    # on the host) and an actor with both a host and a device fire function.
    assert H.validate_demo(4) == 2


def test_cmd_mem_parity(hashes):
    # cmd_mem (proj/src/bench.cpp:491-525): the reference network shapes
    # restated with this library's model types give the reference's Eq. 1
    # totals, pinned by the compiled reference (tests/golden).
    golden = hashes["mem_totals"]
    assert H.memory("motion", "reference", 320, 240, 1) == (5, golden["motion_320x240_r1"])
    assert H.memory("dpd", "reference", period=65536) == (56, golden["dpd_p65536"])
    # The B200 networks: src (2r) + delay self-loop (3*1+1) + sink (2r) tokens
    # for motion; DPD: config (2 x 4 B), in + out planes interleaved (2 x 8 B
    # x period each).
    S = 320 * 240
    for r in (1, 4):
        assert H.memory("motion", "b200", 320, 240, r) == (3, 2 * r * S + 4 * S + 2 * r * S)
    # DPD (batch 1): control (2 x 4 B) + input and output blocks (2 x 8 B x period each).
    assert H.memory("dpd", "b200", period=65536) == (3, 2 * 4 + 2 * (2 * 8 * 65536))
