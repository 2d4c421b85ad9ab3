"""CPU-side checks of the drop-in boundary: libsdb.so loads without a GPU and
exports every function include/sdb.h declares; the product path refuses to run
on CPU tensors (no fallback)."""
import ctypes
import subprocess

import pytest

import paper_1903_05831_b200 as pkg


def test_library_loads_and_exports_header_symbols():
    lb = pkg.lib()
    names = pkg.header_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lb, n)]
    assert not missing, missing


def test_exported_symbols_are_c_abi():
    out = subprocess.run(["nm", "-D", "--defined-only", pkg.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for n in pkg.header_functions():
        assert n in exported, f"{n} not exported with C linkage"


def test_version_and_error_string():
    lb = pkg.lib()
    assert lb.sdb_version() >= 1
    assert isinstance(lb.sdb_last_error(), bytes)


def test_shape_errors_without_gpu():
    """argument validation mirrors conv2d_out_shape (src/tensor.cpp:157-167) and
    needs no device: the ABI rejects bad shapes before touching CUDA."""
    from paper_1903_05831_b200 import simdet as sd
    lb = sd.L()
    rc = lb.sdb_conv_fprop(None, 1, None, None, None, 1, 4, 4, 8, 8, 7, 7, 1, 0, None)
    assert rc == 1 and b"kernel larger" in lb.sdb_last_error()
    rc = lb.sdb_conv_fprop(None, 1, None, None, None, 1, 4, 4, 8, 8, 3, 3, 0, 0, None)
    assert rc == 1
    rc = lb.sdb_conv_fprop(None, 7, None, None, None, 1, 4, 4, 8, 8, 3, 3, 1, 0, None)
    assert rc == 5


def test_no_cpu_fallback():
    torch = pytest.importorskip("torch")
    from paper_1903_05831_b200 import simdet as sd
    with pytest.raises(RuntimeError):
        sd.conv_fprop_nhwc(torch.zeros(1, 4, 4, 8), torch.zeros(8, 3, 3, 8), 1, 1)


def test_error_mapping_matches_reference_taxonomy():
    assert pkg._STATUS[1] is pkg.ShapeError
    assert pkg._STATUS[3] is pkg.DegenerateBatchError
    assert pkg._STATUS[4] is pkg.NonInvertibleError
    with pytest.raises(pkg.ShapeError):
        pkg.check(1)
    assert ctypes.sizeof(ctypes.c_void_p) == 8


def test_checkpoint_plan_matches_reference(ref):
    """sdb_plan_checkpoints == the reference's plan_checkpoints(L)
    (src/memopt.cpp:76-89) for L = 1..200, and PlanError's domain (L < 1)
    is rejected; tests/test_memopt.cpp:88-110 properties hold"""
    import math
    import numpy as np
    lb = pkg.lib()
    lb.sdb_plan_checkpoints.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    for L in range(1, 201):
        starts = np.zeros(64, np.int32)
        S = lb.sdb_plan_checkpoints(L, starts.ctypes.data, 64)
        want = np.zeros(64, np.int64)
        nb = ref.ref_plan_checkpoints(L, want.ctypes.data, 64)
        assert nb >= 0
        assert S == nb + 1 == math.ceil(math.sqrt(L))
        assert starts[0] == 0 and starts[S] == L
        assert list(starts[1:S]) == list(want[:nb])
        seg = np.diff(starts[: S + 1])
        assert seg.min() >= 1 and seg.max() <= (L + S - 1) // S + 1
    assert lb.sdb_plan_checkpoints(0, None, 0) == 5  # SDB_PARAM
    assert ref.ref_plan_checkpoints(0, None, 0) == -1
