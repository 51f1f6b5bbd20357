"""B200 (sm_100a) GPU-actor path of the dynflow dataflow framework
(arXiv 1611.03226).  The product is libdf_cuda.so behind the C ABI in
include/df_cuda.h plus the C++ host runtime in include/df/; this package is
the Python binding used by the tests and bench.py.  No CPU fallback."""
from ._lib import (ControlError, CudaError, DfError, EndOfStream, InvalidArgument, LogicError,  # noqa: F401
                   RunAborted, WatchdogTimeout, LIB_PATH, device_count, header_symbols, lib)

__all__ = ["lib", "device_count", "header_symbols", "LIB_PATH", "DfError", "InvalidArgument",
           "LogicError", "RunAborted", "ControlError", "CudaError", "EndOfStream", "WatchdogTimeout"]
