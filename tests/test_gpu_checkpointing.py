"""sqrt(L) activation checkpointing of the backbone (memory.checkpoint,
src/trainer.cpp:233 -> run_checkpointed_backward, src/memopt.cpp:150-210):
only the segment-boundary block outputs persist, the rest of every segment
lives in one shared arena that backward refills by re-running the segment's
forward from its boundary.  Every kernel is deterministic, so the step must be
BIT-IDENTICAL to the plain one (tests/test_memopt.cpp:112-126: "checkpointed
gradients are bitwise-equal to plain backward"), and the backbone activation
footprint must drop (tests/test_memopt.cpp:139-150)."""
import numpy as np
import pytest

from tests import det_parity as dp

pytestmark = pytest.mark.gpu


def _run(p, steps):
    from paper_1903_05831_b200 import detector as D
    det = D.Detector(p)
    losses = []
    for step in range(1, steps + 1):
        det.feed(D.batch_slots(step, 0, 1, p.batch))
        det.step()
        losses.append(det.losses())
    mem = det.memory()
    w, v = dp.flat_params(det), dp.flat_velocity(det)
    det.close()
    return losses, w, v, mem


@pytest.mark.parametrize("name,kw", [
    ("c1", dict(img_h=128, img_w=128)),                   # fp32 BN+ReLU, L = 3 -> 2 segments
    ("c2", dict(img_h=128, img_w=128)),                   # fp16 IABN, L = 3
    ("c4", dict(img_h=320, img_w=480)),                   # R50-C4: L = 13 -> 4 segments (4, 3, 3, 3)
])
def test_checkpointed_step_is_bit_identical(name, kw):
    from paper_1903_05831_b200 import detector as D
    steps = 2 if name == "c4" else 3
    l0, w0, v0, m0 = _run(D.preset(name, **kw), steps)
    l1, w1, v1, m1 = _run(D.preset(name, extra={"checkpoint": 1}, **kw), steps)
    assert l0 == l1
    assert np.array_equal(w0.view(np.uint32), w1.view(np.uint32))
    assert np.array_equal(v0.view(np.uint32), v1.view(np.uint32))
    L = 13 if name == "c4" else 3
    assert m0[2] == 0 and m1[2] == int(np.ceil(np.sqrt(L)))
    # fewer backbone activation bytes; the device total drops by the same amount
    assert m1[0] < m0[0]
    assert m0[1] - m1[1] == m0[0] - m1[0]
    if name == "c4":
        # the first segment holds all of res2 (the widest maps), so the saving
        # is ~1/3 rather than the uniform chain's 1 - 2/sqrt(L)
        assert m1[0] <= 0.75 * m0[0], (m1[0], m0[0])
