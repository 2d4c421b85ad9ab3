"""The reference-side binding is a real translation unit:
integration/simdet_gpu.cpp compiles against the reference headers
(/root/reference/proj/include: tensor.hpp, syncbn.hpp, memopt.hpp, errors.hpp)
and include/sdb.h, and the built shim library loads, resolving the reference
engine and libsdb.  Argument validation that precedes any device work raises
the reference's own exceptions (conv2d_out_shape's ShapeError) without a GPU."""
import os
import subprocess

import numpy as np
import pytest

from oracle import p
from tests import shim

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists("/root/reference/proj/include/simdet/tensor.hpp"),
                    reason="reference headers absent (GPU box)")
def test_shim_translation_unit_compiles_against_reference_headers():
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "integration"), "check"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.skipif(not shim.available(), reason="shim not built")
def test_shim_loads_and_maps_reference_errors_without_gpu():
    lb = shim.lib()
    for name in shim.SIGS:
        assert hasattr(lb, name)
    x = np.zeros((1, 8, 4, 4), np.float32)
    k = np.zeros((8, 8, 7, 7), np.float32)
    y = np.zeros(64, np.float32)
    # kernel larger than the padded input: simdet::conv2d_out_shape throws ShapeError (status 1)
    assert lb.shim_conv2d(p(x), 1, 8, 4, 4, p(k), 8, 7, 7, 1, 0, 0, p(y)) == 1
    assert b"kernel" in lb.shim_last_error() or len(lb.shim_last_error()) > 0
