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


def test_unknown_channel_is_build_error():
    assert H.validate_demo(3) == -1
    assert b"BuildError" in H.lib().dfh_last_error()


def test_validate_cpu_actor_rules():
    # A dynamic CPU actor (control tokens are consumed on the device, GPU
    # actors only) and an actor with both a host and a device fire function.
    assert H.validate_demo(4) == 2
