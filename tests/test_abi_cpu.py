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
