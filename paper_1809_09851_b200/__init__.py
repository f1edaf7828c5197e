"""B200-native evaluation backend for the fusevec (arXiv 1809.09851) hot path.

The product is ``lib/libfvb.so`` (sm_100a kernels behind the C ABI in
``include/fvb.h``).  This package only loads it and offers thin typed
wrappers over torch CUDA tensors for tests and the benchmark; there is no
CPU fallback -- a missing or unloadable library raises immediately.
"""

from ._native import (  # noqa: F401
    ArgumentError,
    DeviceError,
    FvbError,
    LengthMismatch,
    PrecisionError,
    UnsupportedExpression,
    lib,
    lib_path,
)
from .device import (  # noqa: F401
    DEFAULT_GAS,
    Gas,
    HostContext,
    axpy_sin,
    cons2prim,
    csr_matvec_acc,
    emit_source,
    eos,
    flux,
    flux_prim,
    jacobian,
    lookup,
    nvrtc_compile,
    patterns,
    prim2cons,
    synth_state,
    synth_uniform,
    v_mag2,
    wave_speed_max,
)

__all__ = [name for name in dir() if not name.startswith("_")]
