"""Pin the CPU restatement against golden vectors generated from the compiled
reference engine (tests/golden/make_golden.py) -- runs without the reference."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import p

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_half_rounding(orc, gold):
    v = gold["half_in"]
    want = gold["half_bits"].view(np.float16).astype(np.float32)
    got = np.zeros_like(v)
    orc.orc_half_round_n(p(v), p(got), v.size)
    assert np.array_equal(np.nan_to_num(got).view(np.uint32), np.nan_to_num(want).view(np.uint32))


@pytest.mark.parametrize("seed", range(6))
def test_nms_keep_lists(orc, gold, seed):
    boxes = gold[f"nms{seed}_boxes"]
    scores = gold[f"nms{seed}_scores"]
    n = len(scores)
    order = np.zeros(n, np.int32)
    orc.orc_topk_order(p(scores), n, n, p(order))
    sb = np.ascontiguousarray(boxes[order])
    keep = np.zeros(n, np.int32)
    k = orc.orc_nms_sorted(p(sb), n, 0.5, n, p(keep))
    assert list(order[keep[:k]]) == list(gold[f"nms{seed}_keep"])


def test_update_scale_trace(orc, gold):
    s, g = C.c_double(32768.0), C.c_int64(0)
    for o, (ws, wg) in zip(gold["scale_overflow"], gold["scale_trace"]):
        orc.orc_update_scale(C.byref(s), C.byref(g), 1, 13, 2.0, 0.5, 1.0, 2.0**20, int(o))
        assert (s.value, g.value) == (ws, wg)


def test_sgd_step(orc, gold):
    w, v, g = gold["sgd_w0"].copy(), gold["sgd_v0"].copy(), gold["sgd_g"]
    orc.orc_apply_sgd(p(w), p(v), p(g), w.size, 0.01, 0.9, 1.0)
    assert np.array_equal(w.view(np.uint32), gold["sgd_w1"].view(np.uint32))
    assert np.array_equal(v.view(np.uint32), gold["sgd_v1"].view(np.uint32))
