"""The data-parallel code path on ONE GPU (no second device is available to
this suite): a forced 1-rank NCCL communicator makes the step issue exactly
what it issues at K > 1 -- per-bucket split-K reduces on the wgrad stream, a
bucket allreduce (ncclAvg over fp16) on the comm stream for each bucket, the
fp32 BN-gradient and f64 loss allreduces -- inside the captured CUDA graph.
At K = 1 every collective is an identity, so the step must be BIT-IDENTICAL
to the plain step (src/trainer.cpp:240-257 order), whatever the bucket plan.
Reference: CommGroup::allreduce_sum (src/comm.cpp:288-315), the step tail
(src/trainer.cpp:240-257), the injected-overflow trajectory
(tests/test_trainer.cpp:292-321)."""
import numpy as np
import pytest

from tests import det_parity as dp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _run(p, steps, force_comm, poison_at=None):
    from paper_1903_05831_b200 import detector as D
    det = D.Detector(p, force_comm=force_comm)
    traj = []
    for step in range(1, steps + 1):
        if poison_at == step:
            w = det.get_param(0)
            w.flat[0] = np.inf
            det.set_param(0, w)
        det.feed(D.batch_slots(step, 0, 1, p.batch))
        det.step()
        losses, scale, ov = det.losses()
        traj.append((losses, scale, ov))
        if poison_at == step:  # repair the weight, as a restarted run would
            w = det.get_param(0)
            w.flat[0] = 0.0
            det.set_param(0, w)
    w = dp.flat_params(det)
    v = dp.flat_velocity(det)
    det.close()
    return traj, w, v


@pytest.mark.parametrize("shard", [1, 0])
@pytest.mark.parametrize("bucket_mb", [25.0, 0.05])
def test_forced_comm_step_is_bit_identical(bucket_mb, shard):
    """4 steps (1 eager + 3 graph replays) with the comm path on == the plain
    step, bit for bit; bucket_mb 0.05 splits the tiny detector into dozens of
    buckets, so bucket completion order and per-bucket reduces are exercised.
    shard = 1: reduce-scatter + per-shard update + all-gather of the fp16
    shadows; shard = 0: bucket allreduce + replicated update"""
    from paper_1903_05831_b200 import detector as D
    p = D.preset("c2", img_h=128, img_w=128, extra={"bucket_mb": bucket_mb, "shard_optimizer": shard})
    t0, w0, v0 = _run(p, 4, False)
    t1, w1, v1 = _run(p, 4, True)
    assert [t[0] for t in t0] == [t[0] for t in t1]
    assert np.array_equal(w0.view(np.uint32), w1.view(np.uint32))
    assert np.array_equal(v0.view(np.uint32), v1.view(np.uint32))


def test_bucket_plan_does_not_change_the_step():
    """the per-bucket reduce schedule is a pure regrouping of the split-K jobs"""
    from paper_1903_05831_b200 import detector as D
    base = D.preset("c2", img_h=128, img_w=128)
    _, wa, _ = _run(base, 3, False)
    _, wb, _ = _run(D.preset("c2", img_h=128, img_w=128, extra={"bucket_mb": 0.02}), 3, False)
    assert np.array_equal(wa.view(np.uint32), wb.view(np.uint32))


def test_dynamic_scale_trajectory_with_injected_overflow(ref):
    """C5's dynamic loss scale (growth every N clean steps, x0.5 on overflow)
    through the comm path: the scale used per step and the skip flags follow the
    reference update_scale (src/precision.cpp:45-56) over an injected overflow,
    and the skipped step leaves weights and velocity untouched
    (tests/test_trainer.cpp:292-321)"""
    import ctypes as C
    from paper_1903_05831_b200 import detector as D
    p = D.preset("c2", img_h=128, img_w=128, dynamic_scale=1, scale_init=2.0**15, growth_interval=2)
    traj, _, _ = _run(p, 7, True, poison_at=4)
    flags = [t[2] for t in traj]
    assert flags == [0, 0, 0, 1, 0, 0, 0]
    # reference state machine over the same overflow sequence
    s, good = C.c_double(2.0**15), C.c_int64(0)
    want = []
    for ov in flags:
        want.append(s.value)
        assert ref.ref_update_scale(C.byref(s), C.byref(good), 1, 2, 2.0, 0.5, 1.0, 16777216.0, ov) == 0
    assert [t[1] for t in traj] == want


def test_allreduce_abi_on_one_rank():
    """sdb_allreduce_sum on a 1-rank communicator is the identity (f16/f32/f64),
    and the watchdog reports no asynchronous error"""
    import ctypes as C
    from paper_1903_05831_b200 import detector as D
    from paper_1903_05831_b200 import simdet as sd
    lb = D.L()
    buf = C.create_string_buffer(128)
    assert lb.sdb_get_nccl_unique_id(buf) == 0
    h = C.c_void_p()
    assert sd.L().sdb_ctx_create(0, 0, 1, buf, C.byref(h)) == 0
    try:
        for dtp in (torch.float16, torch.float32, torch.float64):
            x = torch.randn(1000003, device="cuda").to(dtp)
            y = x.clone()
            sd.allreduce_sum(y, context=h)
            torch.cuda.synchronize()
            assert torch.equal(x, y)
        assert sd.L().sdb_comm_check(h) == 0
    finally:
        sd.L().sdb_ctx_destroy(h)


@pytest.mark.parametrize("force_comm", [False, True])
def test_sync_bn_mode_on_one_rank_is_plain_bn(force_comm):
    """bn.mode "sync" (src/model.cpp:204): every BN layer's float [sum, sumsq,
    count] and backward [sum dy, sum dy*xhat] go through an fp32 SUM allreduce
    on the step stream (src/syncbn.cpp:21-117).  On one rank the reference skips
    the allreduce (group->size() > 1) and so the step equals plain BN
    bit for bit; with the forced 1-rank communicator the NCCL calls run inside
    the captured step and must not change a bit either.  The K > 1 sums are
    pinned on CPU (tests/test_oracle_pins.py: the restatement vs the reference's
    own run_workers groups)."""
    from paper_1903_05831_b200 import detector as D
    base = D.preset("c1", img_h=128, img_w=128)
    t0, w0, v0 = _run(base, 3, False)
    t1, w1, v1 = _run(D.preset("c1", img_h=128, img_w=128, extra={"sync_bn": 1}), 3, force_comm)
    assert [t[0] for t in t0] == [t[0] for t in t1]
    assert np.array_equal(w0.view(np.uint32), w1.view(np.uint32))
    assert np.array_equal(v0.view(np.uint32), v1.view(np.uint32))


def test_sync_bn_needs_bn_mode():
    from paper_1903_05831_b200 import ParamError
    from paper_1903_05831_b200 import detector as D
    with pytest.raises(ParamError):
        D.Detector(D.preset("c2", img_h=128, img_w=128, extra={"sync_bn": 1}))


def test_concurrent_shortcut_branch_is_bit_identical(monkeypatch):
    """the downsampling blocks' shortcut (down conv + its InPlace-ABN) runs on a
    second stream next to conv1-conv3 inside the captured step; the step must
    not change a bit against the sequential schedule (SDB_NO_BRANCH)"""
    from paper_1903_05831_b200 import detector as D
    p = D.preset("c2", img_h=128, img_w=128)
    t0, w0, v0 = _run(p, 3, False)
    monkeypatch.setenv("SDB_NO_BRANCH", "1")
    t1, w1, v1 = _run(p, 3, False)
    assert [t[0] for t in t0] == [t[0] for t in t1]
    assert np.array_equal(w0.view(np.uint32), w1.view(np.uint32))
    assert np.array_equal(v0.view(np.uint32), v1.view(np.uint32))



@pytest.mark.parametrize("steps", [3])
def test_head_pool_fusion_is_bit_identical(monkeypatch, steps):
    """the last RoI-head block's apply pass average-pools the block output
    itself (not stored; the backward masks with its sign bitmap): the step
    must equal the separate avgpool_fwd / masked avgpool_bwd bit for bit
    (SDB_NO_HEAD_POOL_FUSE)"""
    from paper_1903_05831_b200 import detector as D
    p = D.preset("c5", img_h=160, img_w=224)
    det = D.Detector(p)
    with pytest.raises(Exception):  # the fused path is the one under test: head_out is not stored
        det.export(19, np.float16)
    det.close()
    t0, w0, v0 = _run(p, steps, False)
    monkeypatch.setenv("SDB_NO_HEAD_POOL_FUSE", "1")
    t1, w1, v1 = _run(p, steps, False)
    assert [t[0] for t in t0] == [t[0] for t in t1]
    assert np.array_equal(w0.view(np.uint32), w1.view(np.uint32))
    assert np.array_equal(v0.view(np.uint32), v1.view(np.uint32))
