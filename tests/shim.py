"""TEST INFRASTRUCTURE: ctypes bindings of the reference-side shim veneer
(integration/_build/libsimdet_gpu_shim.so = integration/simdet_gpu.cpp, the
simdet::gpu translation unit of INTEGRATION.md, + shim_check.cpp)."""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SHIM_PATH = os.path.join(os.path.dirname(HERE), "integration", "_build", "libsimdet_gpu_shim.so")
_P, _I, _L, _F, _D = C.c_void_p, C.c_int, C.c_int64, C.c_float, C.c_double
SIGS = {
    "shim_last_error": (C.c_char_p, []),
    "shim_conv2d": (_I, [_P, _I, _I, _I, _I, _P, _I, _I, _I, _I, _I, _I, _P]),
    "shim_conv2d_backward": (_I, [_P, _I, _I, _I, _I, _P, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    "shim_bn_forward": (_I, [_P, _I, _I, _I, _I, _P, _P, _F, _I, _P, _P, _P, _P, _P, _P]),
    "shim_bn_backward": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P]),
    "shim_iabn_forward": (_I, [_P, _I, _I, _I, _I, _P, _P, _F, _F, _I, _P, _P, _P]),
    "shim_iabn_backward": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _F, _F, _I, _P, _P, _P]),
    "shim_apply_sgd": (_I, [_P, _P, _P, _L, _F, _F, _D, _I, _P]),
}
_lib = None


def available():
    return os.path.exists(SHIM_PATH)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(SHIM_PATH)
        for n, (res, args) in SIGS.items():
            f = getattr(_lib, n)
            f.restype, f.argtypes = res, args
    return _lib
