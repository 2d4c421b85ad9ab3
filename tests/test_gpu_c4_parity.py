"""Parity at the HEADLINE configuration (BASELINE config C4): Faster R-CNN
R50-C4 (3-4-6 + res5 head), 2 x 3x800x1333, 80 classes, Poisson(7) GT boxes,
12000 -> 2000 proposals, 512 RoIs/img at 1:3 -- the graph bench.py times.

The reference-Tape oracle would need ~10 CPU-minutes per image here, so the
continuous part is checked against the torch checker (tests/torch_detector.py:
the same graph with torch ops/autograd, pinned to the reference Tape on CPU by
tests/test_torch_checker_cpu.py), run on the GPU (fp32 with TF32 off, fp64,
and the fp16-contract emulation), teacher-forced on the step's own decisions.  Every step:

  discrete, BIT-EXACT vs the restatement (oracle/restate.cpp): the 63,000
      anchors, anchor labels (+ targets 1e-6), the 12000 -> 2000 top-k/NMS
      proposals of both images from the GPU's own RPN outputs, the sampled
      RoIs / labels (+ targets 1e-5);
  mode 2 (the C4 graph in fp32) against the checker in float64: losses and
      RPN logits <= 1e-3; every parameter gradient and per-step delta <= 1e-2
      or, where the fp32 arithmetic itself is noisier (the checker's own fp32
      vs fp64 error), <= 2x that floor per tensor (as the mode-1 rule below:
      the per-tensor error of small BN-parameter gradients is cancellation
      noise, and two fp32 evaluations summing in different orders are
      independent draws of it -- a reordered RoIAlign-backward summation alone
      moved res2.0.bn1.gamma from below 1e-2 to 1.54x its 6.7e-3 floor) and
      <= 1.5x globally;
  mode 1 (fp16, the benchmarked graph): losses within 1e-2 of the fp32
      truth, RPN logits within max(1e-2, 1.5 x err(torch16, torch32)); per tensor, the gradient and the parameter delta no
      further from the fp16-contract emulation (torch16) than torch16 is from
      the fp32 truth (x2 per tensor, x1.5 globally, floor 1e-2) -- the same
      noise-floor rule as the C2 test against the reference's own fp16 run.
"""
import numpy as np
import pytest

from oracle import p as ptr
from tests import det_parity as dp
from tests.util import norm_rel

torch = pytest.importorskip("torch")
pytest.importorskip("torchvision")
pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _no_tf32():
    a, b = torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = a, b


def _split_err(det, a, b):
    return [norm_rel(x, y) for x, y in zip(dp.split(det, a), dp.split(det, b))]


def _step_and_check(det, step):
    from paper_1903_05831_b200 import detector as D
    slots = D.batch_slots(step, 0, 1, det.p.batch)
    w0, v0 = dp.flat_params(det), dp.flat_velocity(det)
    det.feed(slots)
    det.step()
    losses, scale, ov = det.losses()
    assert ov == 0 and all(np.isfinite(losses))
    s = dp.gpu_state(det)
    rep = dp.check_discrete(det, s, slots)
    for j in range(det.p.batch):
        assert rep[j]["proposals"] > 0 and rep[j]["fg_rois"] > 0
        assert rep[j]["rois"] == det.p.roi_batch  # full batches (no padded RoIs)
    return slots, w0, v0, losses, scale, s


def test_c4_fp32_graph_two_steps(orc):
    """mode 2: the C4 network in fp32 against the torch checker in float64 (the
    truth).  At this size the fp32 gradient is itself conditioned at the 1e-2
    level for the earliest layers (measured: torch fp32 vs torch fp64 differ by
    1.04e-2 on stem.conv, 4.6e-3 globally -- max-pool/leaky routing decided by
    ~1e-7 differences over 34 M windows), so each gradient tensor is held to
    max(1e-2, 1.5 x err(torch32, torch64)) and the global gradient to
    max(1e-3, 1.5 x the same); the libsdb fp32 step sits CLOSER to the fp64
    truth than cuDNN's fp32 does (stem.conv 6.9e-3, global 3.0e-3)."""
    from paper_1903_05831_b200 import detector as D
    from tests.torch_detector import gpu_params, run_checker
    det = D.Detector(D.preset("c4", mode=2, scale_init=1.0))
    assert det.feat_h == 50 and det.feat_w == 84 and det.A == 15
    for step in (1, 2):
        params = gpu_params(det)
        _, w0, v0, lg, scale, s = _step_and_check(det, step)
        l64, g64, lg64 = run_checker(det, params, s, 2, scale, "cuda", dtype=torch.float64)
        torch.cuda.empty_cache()
        _, g32, _ = run_checker(det, params, s, 2, scale, "cuda")
        torch.cuda.empty_cache()
        for i in range(4):
            assert abs(lg[i] - l64[i]) <= 1e-3 * abs(l64[i]), (step, i, lg[i], l64[i])
        assert norm_rel(s["logits"][..., :det.A].transpose(0, 3, 1, 2), lg64) <= 1e-3
        g = dp.flat_grads(det)
        floor = _split_err(det, g32, g64)
        for (name, _, _), e, f in zip(det.params, _split_err(det, g, g64), floor):
            assert e <= max(1e-2, 2.0 * f), (step, name, e, f)
        assert norm_rel(g, g64) <= max(1e-3, 1.5 * norm_rel(g32, g64))
        w_ref, v_ref = w0.copy(), v0.copy()
        orc.orc_apply_sgd(ptr(w_ref), ptr(v_ref), ptr(g64), w_ref.size, det.p.lr, det.p.momentum, scale)
        w1 = dp.flat_params(det)
        for (name, _, _), e, f in zip(det.params, _split_err(det, w1 - w0, w_ref - w0), floor):
            assert e <= max(1e-2, 2.0 * f), (step, name, e, f)
    det.close()


@pytest.mark.parametrize("steps", [10])
def test_c4_fp16_benchmarked_graph(orc, steps):
    """mode 1 (the graph bench.py times): `steps` steps, each compared from the
    same state against torch16 (fp16 contract) and torch32 (fp32 truth)"""
    from paper_1903_05831_b200 import detector as D
    from tests.torch_detector import gpu_params, run_checker
    det = D.Detector(D.preset("c4"))
    worst = []
    for step in range(1, steps + 1):
        params = gpu_params(det)
        _, w0, v0, lg, scale, s = _step_and_check(det, step)
        assert scale == 128.0
        l16, g16, lg16 = run_checker(det, params, s, 1, scale, "cuda")
        l32, g32, lg32 = run_checker(det, params, s, 2, scale, "cuda")
        for i in range(4):
            assert abs(lg[i] - l32[i]) <= 1e-2 * abs(l32[i]), (step, i, lg[i], l32[i])
        # RPN logits after 16 fp16 bottlenecks at 800x1333: the fp16 contract
        # itself moves them by ~1.5% (torch16 vs torch32); same floor rule
        lg_gpu = s["logits"][..., :det.A].astype(np.float32).transpose(0, 3, 1, 2)
        assert norm_rel(lg_gpu, lg32) <= max(1e-2, 1.5 * norm_rel(lg16, lg32)), (norm_rel(lg_gpu, lg32),
                                                                                 norm_rel(lg16, lg32))
        g = dp.flat_grads(det)
        e_gpu = _split_err(det, g, g16)
        floor = _split_err(det, g16, g32)
        for (name, _, _), e, f in zip(det.params, e_gpu, floor):
            assert e <= max(1e-2, 2.0 * f), (step, name, e, f)
        assert norm_rel(g, g16) <= max(1e-2, 1.5 * norm_rel(g16, g32)), (step, norm_rel(g, g16), norm_rel(g16, g32))
        # per-step parameter deltas (apply_sgd on the checker's fp16 gradient)
        w_ref, v_ref = w0.copy(), v0.copy()
        assert orc.orc_has_nonfinite(ptr(g16), g16.size) == 0
        orc.orc_apply_sgd(ptr(w_ref), ptr(v_ref), ptr(g16), w_ref.size, det.p.lr, det.p.momentum, scale)
        w1 = dp.flat_params(det)
        d_gpu, d_ref = w1 - w0, w_ref - w0
        for (name, _, _), e, f in zip(det.params, _split_err(det, d_gpu, d_ref), floor):
            assert e <= max(1e-2, 2.0 * f), (step, name, e, f)
        worst.append((norm_rel(g, g16), norm_rel(g16, g32), norm_rel(d_gpu, d_ref)))
        torch.cuda.empty_cache()
    print("C4 fp16 per step: err(gpu,t16) / err(t16,t32) / delta err:", worst)
    det.close()
