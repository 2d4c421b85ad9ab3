"""paper_1903_05831_b200 -- B200-native (sm_100a) SimpleDet Faster R-CNN C4
training step behind the reference engine's operator API.

The compute lives in ``libsdb.so`` (hand-written CUDA for sm_100a + C++ host
driver, C ABI in ``include/sdb.h``).  This module only loads it with ctypes and
exposes (a) the raw ABI and (b) a thin host mirror of the reference's C++
operator API (``simdet.py``).  There is NO CPU fallback: importing the ops
without the built library, or calling them without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
# SDB_LIB: diagnostic override (A/B of two builds, tools/step_digest.py)
LIB_PATH = os.environ.get("SDB_LIB") or os.path.join(_HERE, "libsdb.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "sdb.h")

F32 = 0
F16 = 1

_lib = None


class SdbError(RuntimeError):
    """Base of the mirrored reference exception taxonomy (errors.hpp:9-40)."""


class ShapeError(SdbError):
    pass


class ContractError(SdbError):
    pass


class DegenerateBatchError(SdbError):
    pass


class NonInvertibleError(SdbError):
    pass


class ParamError(SdbError):
    pass


class CollectiveError(SdbError):
    pass


class CudaError(SdbError):
    pass


class UnsupportedError(SdbError):
    pass


class FormatError(SdbError):
    pass


class ConfigError(SdbError):
    """simdet::ConfigError (errors.hpp:37): raised by the training driver, not the ABI"""


_STATUS = {1: ShapeError, 2: ContractError, 3: DegenerateBatchError, 4: NonInvertibleError, 5: ParamError,
           6: CollectiveError, 7: CudaError, 8: UnsupportedError, 9: FormatError}


def header_functions() -> list[str]:
    """Names of every function declared in include/sdb.h."""
    src = open(HEADER_PATH).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sdb_[a-z0-9_]+)\s*\(", src)))


def lib() -> ctypes.CDLL:
    """Load libsdb.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        _lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        _lib.sdb_last_error.restype = ctypes.c_char_p
        _lib.sdb_ctx_stream.restype = ctypes.c_void_p
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().sdb_last_error().decode(errors="replace")
        raise _STATUS.get(rc, SdbError)(msg)
