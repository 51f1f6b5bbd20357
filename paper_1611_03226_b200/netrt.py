"""ctypes view of the device-resident network runtime (df_net_*, csrc/netrt.cu).

Test/bench harness only: it builds networks of the library's device actor
kinds over device channels and runs them as one persistent kernel.  All the
work happens in libdf_cuda.so; nothing here computes."""
from __future__ import annotations

import ctypes as C

from ._lib import call, lib

DF_ACT_DPD_SOURCE, DF_ACT_DPD_CONFIG, DF_ACT_DPD_SPLIT, DF_ACT_DPD_BRANCH, DF_ACT_DPD_ADDER, DF_ACT_DPD_SINK = range(1, 7)
DF_ACT_TEST_PRODUCE, DF_ACT_TEST_CONSUME = 7, 8
DF_ACT_FRAME_SOURCE, DF_ACT_GAUSS, DF_ACT_THRES, DF_ACT_MEDIAN, DF_ACT_FRAME_SINK = range(9, 14)


class Samples(C.Structure):
    _fields_ = [("samples", C.c_void_p), ("period", C.c_uint32)]


class Config(C.Structure):
    _fields_ = [("schedule", C.c_void_p), ("len", C.c_uint32)]


class Branch(C.Structure):
    _fields_ = [("branch", C.c_uint32), ("taps_per_branch", C.c_uint32), ("taps", C.c_void_p),
                ("state", C.c_void_p), ("period", C.c_uint32)]


class Test(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("counters", C.c_void_p), ("stall_mask", C.c_uint32),
                ("skip_initial", C.c_uint32), ("hold_ns", C.c_uint64)]


class Frames(C.Structure):
    _fields_ = [("frames", C.c_void_p), ("width", C.c_uint32), ("height", C.c_uint32), ("threshold", C.c_uint8)]


class Net:
    """df_net: add actors (kind, params, ctas, control, inputs, outputs,
    firing limit), optional control tables, then run() once."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        call("df_net_create", device, C.byref(h))
        self.handle = h

    def add(self, kind: int, params=None, ctas: int = 1, control=None, inputs=(), outputs=(), limit: int = 0) -> int:
        ins = (C.c_void_p * max(1, len(inputs)))(*[c.handle for c in inputs])
        outs = (C.c_void_p * max(1, len(outputs)))(*[c.handle for c in outputs])
        idx = C.c_int(-1)
        call("df_net_add_actor", self.handle, kind, C.byref(params) if params is not None else None,
             C.sizeof(params) if params is not None else 0, ctas, control.handle if control else None,
             ins, len(inputs), outs, len(outputs), limit, C.byref(idx))
        return idx.value

    def control_table(self, actor: int, rows):
        """rows: one (in_bits, out_bits, legal) triple per token value."""
        flat = (C.c_uint32 * (3 * len(rows)))(*[int(v) for r in rows for v in r])
        call("df_net_set_control_table", self.handle, actor, flat, len(rows))

    def run(self, timeout_s: float = 10.0):
        call("df_net_run", self.handle, float(timeout_s))

    def abort(self):
        call("df_net_abort", self.handle)

    def fault(self):
        a, c, t = C.c_int(), C.c_int(), C.c_uint32()
        call("df_net_fault", self.handle, C.byref(a), C.byref(c), C.byref(t))
        return a.value, c.value, t.value

    def stats(self, actor: int):
        f, ms = C.c_uint64(), C.c_double()
        call("df_net_actor_stats", self.handle, actor, C.byref(f), C.byref(ms))
        return f.value, ms.value

    def profile(self, actor: int):
        """(wait_ms, fire_ms, commit_ms) of the actor's leader over the run."""
        w, f, c = C.c_double(), C.c_double(), C.c_double()
        call("df_net_actor_profile", self.handle, actor, C.byref(w), C.byref(f), C.byref(c))
        return w.value, f.value, c.value

    def close(self):
        if self.handle:
            lib().df_net_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
