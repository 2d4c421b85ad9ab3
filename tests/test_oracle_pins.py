"""Pin the CPU restatement (oracle/restate.cpp) to the reference: against the
compiled reference engine (oracle/_ref) and against the golden vectors of the
reference's own tests (tests/test_half.cpp, test_precision.cpp,
test_postproc.cpp under /root/reference/proj)."""
import ctypes as C

import numpy as np
import pytest

import oracle
from oracle import p


# ---------------------------------------------------------------- binary16
def test_half_golden_vectors(orc):
    # tests/test_half.cpp:52-72
    assert orc.orc_half_round(65504.0) == 65504.0
    assert np.isinf(orc.orc_half_round(65520.0))
    assert orc.orc_half_round(2.0**-25) == 0.0
    assert orc.orc_half_round(1.0 + 2.0**-11) == 1.0
    assert np.signbit(orc.orc_half_round(-0.0))


def test_half_matches_reference_bits(orc, ref):
    rng = np.random.default_rng(0)
    vals = np.concatenate([
        rng.standard_normal(20000).astype(np.float32) * 1e3,
        (rng.random(20000) * 2.0**-14).astype(np.float32),
        np.array([65504, 65519.99, 65520, 1e-8, 2**-24, 3 * 2**-26, -2**-25], np.float32),
    ])
    for v in vals:
        r = ref.ref_half_bits_to_float(ref.ref_float_to_half_bits(float(v)))
        o = orc.orc_half_round(float(v))
        assert np.float32(r).view(np.uint32) == np.float32(o).view(np.uint32), v


# ---------------------------------------------------------------- loss scale
def test_update_scale_golden_and_reference(orc, ref):
    # tests/test_precision.cpp:24-54: overflow halves 1024 -> 512
    s, g = C.c_double(1024.0), C.c_int64(5)
    orc.orc_update_scale(C.byref(s), C.byref(g), 1, 2000, 2.0, 0.5, 1.0, 2.0**24, 1)
    assert s.value == 512.0 and g.value == 0
    rng = np.random.default_rng(1)
    for trial in range(20):
        s1, g1, s2, g2 = C.c_double(2.0**15), C.c_int64(0), C.c_double(2.0**15), C.c_int64(0)
        for ov in (rng.random(300) < 0.05 * (trial % 4)):
            orc.orc_update_scale(C.byref(s1), C.byref(g1), 1, 9, 2.0, 0.5, 1.0, 2.0**17, int(ov))
            ref.ref_update_scale(C.byref(s2), C.byref(g2), 1, 9, 2.0, 0.5, 1.0, 2.0**17, int(ov))
            assert (s1.value, g1.value) == (s2.value, g2.value)
    # static mode is a no-op
    s = C.c_double(128.0)
    orc.orc_update_scale(C.byref(s), C.byref(g), 0, 9, 2.0, 0.5, 1.0, 2.0**17, 1)
    assert s.value == 128.0


# ---------------------------------------------------------------- optimizer
def test_apply_sgd_two_step_closed_form(orc):
    # tests/test_precision.cpp:115-127: g = 1 twice -> w2 = w0 - lr - lr(mu+1)
    w = np.array([1.0], np.float32)
    v = np.zeros(1, np.float32)
    g = np.ones(1, np.float32)
    for _ in range(2):
        orc.orc_apply_sgd(p(w), p(v), p(g), 1, 0.1, 0.9, 1.0)
    expect = np.float32(1.0) - np.float32(0.1) - np.float32(0.1) * np.float32(1.9)
    assert abs(w[0] - expect) < 1e-6


def test_apply_sgd_equals_reference_master_step(orc, ref):
    # with denom == 1 apply_sgd reduces to sgd_step_master (src/precision.cpp:84-100)
    rng = np.random.default_rng(2)
    n = 4099
    w = rng.standard_normal(n).astype(np.float32)
    v = rng.standard_normal(n).astype(np.float32) * 0.1
    g = rng.standard_normal(n).astype(np.float32)
    w1, v1, w2, v2 = w.copy(), v.copy(), w.copy(), v.copy()
    orc.orc_apply_sgd(p(w1), p(v1), p(g), n, 0.01, 0.9, 1.0)
    assert ref.ref_sgd_step_master(p(w2), p(v2), p(g), n, 0.01, 0.9) == 0
    assert np.array_equal(w1.view(np.uint32), w2.view(np.uint32))
    assert np.array_equal(v1.view(np.uint32), v2.view(np.uint32))


def test_has_nonfinite(orc):
    a = np.ones(10, np.float32)
    assert orc.orc_has_nonfinite(p(a), 10) == 0
    a[3] = np.inf
    assert orc.orc_has_nonfinite(p(a), 10) == 1


# ---------------------------------------------------------------- IoU / NMS
def _box(*v):
    return np.array(v, np.float32)


def test_iou_golden(orc, ref):
    # tests/test_postproc.cpp:45-56
    a, b = _box(0, 0, 10, 10), _box(5, 5, 15, 15)
    assert abs(orc.orc_iou(p(a), p(b)) - 1.0 / 7.0) < 1e-12
    ad, bd = a.astype(np.float64), b.astype(np.float64)
    assert orc.orc_iou(p(a), p(b)) == ref.ref_iou(p(ad), p(bd))
    z = _box(1, 1, 1, 1)
    assert orc.orc_iou(p(z), p(z)) == 0.0


def test_nms_trio_golden(orc):
    # tests/test_postproc.cpp:58-67: trio IoU 81/119; t=0.5 keeps {0,2}; t=0.7 keeps all
    boxes = np.array([[0, 0, 10, 10], [1, 1, 11, 11], [20, 20, 30, 30]], np.float32)
    assert abs(orc.orc_iou(p(boxes[0]), p(boxes[1])) - 81.0 / 119.0) < 1e-12
    keep = np.zeros(3, np.int32)
    k = orc.orc_nms_sorted(p(boxes), 3, 0.5, 10, p(keep))
    assert list(keep[:k]) == [0, 2]
    k = orc.orc_nms_sorted(p(boxes), 3, 0.7, 10, p(keep))
    assert list(keep[:k]) == [0, 1, 2]


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("thr", [0.3, 0.5, 0.7])
def test_nms_matches_reference(orc, ref, seed, thr):
    """orc_nms_sorted over the (score desc, index asc) order == reference
    nms_greedy (src/postproc.cpp:47-63), bit-exact keep lists."""
    rng = np.random.default_rng(seed)
    n = 300
    xy = rng.random((n, 2)) * 200
    wh = np.exp(rng.uniform(np.log(4), np.log(80), (n, 2)))
    boxes = np.concatenate([xy, xy + wh], 1).astype(np.float32)
    scores = np.round(rng.random(n), 2).astype(np.float32)  # many ties
    order = np.zeros(n, np.int32)
    orc.orc_topk_order(p(scores), n, n, p(order))
    sb = np.ascontiguousarray(boxes[order])
    keep = np.zeros(n, np.int32)
    k = orc.orc_nms_sorted(p(sb), n, thr, n, p(keep))
    mine = list(order[keep[:k]])
    bd = boxes.astype(np.float64)
    sd = scores.astype(np.float64)
    rk = np.zeros(n, np.int64)
    nk = C.c_int64(0)
    assert ref.ref_nms_greedy(p(bd), p(sd), None, n, thr, p(rk), C.byref(nk)) == 0
    assert mine == list(rk[:nk.value])


def test_topk_order_ties_break_low_index(orc):
    s = np.array([0.5, 0.9, 0.5, np.nan, 0.9, -np.inf], np.float32)
    o = np.zeros(6, np.int32)
    orc.orc_topk_order(p(s), 6, 6, p(o))
    assert list(o) == [1, 4, 0, 2, 5, 3]


def test_mix64_matches_reference_dataset_rng(orc):
    # mix64 (src/dataset.cpp:11-17); splitmix64 first output for seed 0 is a
    # well-known constant: next() of state 0 -> 0xe220a8397b1dcdaf
    assert orc.orc_mix64(0, 0) == 0xE220A8397B1DCDAF


# ---------------------------------------------------------------- SyncBN over K ranks
def _shards(K, N, Cc, H, W, fp16, seed):
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((K, N, Cc, H, W)) * 1.7 + 0.3).astype(np.float32)
    dy = rng.standard_normal((K, N, Cc, H, W)).astype(np.float32)
    if fp16:
        x = x.astype(np.float16).astype(np.float32)
        dy = dy.astype(np.float16).astype(np.float32)
    g = (rng.random(Cc) + 0.5).astype(np.float32)
    b = (rng.standard_normal(Cc) * 0.1).astype(np.float32)
    return x, dy, g, b


@pytest.mark.parametrize("K", [1, 2, 3, 4])
@pytest.mark.parametrize("fp16", [0, 1])
def test_syncbn_k_ranks_restatement_matches_reference(orc, ref, K, fp16):
    """syncbn_forward/backward with a K-rank group (src/syncbn.cpp:21-117 over
    the ring allreduce of src/comm.cpp:288-315), reference run_workers vs the
    restatement: bit-identical outputs, statistics and gamma/beta gradients"""
    N, Cc, H, W = 2, 24, 5, 7
    x, dy, g, b = _shards(K, N, Cc, H, W, fp16, 10 * K + fp16)
    outs = {}
    for name, lib in (("orc", orc), ("ref", ref)):
        y = np.zeros_like(x)
        mean, inv = np.zeros(Cc, np.float32), np.zeros(Cc, np.float32)
        agg = np.zeros(2 * Cc + 1, np.float32)
        fn = lib.orc_syncbn_forward_k if name == "orc" else lib.ref_syncbn_forward_k
        rc = fn(K, p(x), N, Cc, H, W, p(g), p(b), 1e-5, fp16, p(y), p(mean), p(inv), p(agg))
        assert not rc
        count = int(agg[2 * Cc])
        dx = np.zeros_like(x)
        dg, db = np.zeros(Cc, np.float32), np.zeros(Cc, np.float32)
        if name == "orc":
            lib.orc_syncbn_backward_k(K, p(dy), p(x), N, Cc, H, W, p(g), p(mean), p(inv), count, p(dx), p(dg), p(db))
        else:
            assert not lib.ref_syncbn_backward_k(K, p(dy), p(x), N, Cc, H, W, p(g), p(mean), p(inv), count, fp16,
                                                 p(dx), p(dg), p(db))
        outs[name] = (y, mean, inv, agg, dx, dg, db)
    for a, r in zip(outs["orc"], outs["ref"]):
        assert np.array_equal(a.view(np.uint32), r.view(np.uint32))
    assert int(outs["ref"][3][2 * Cc]) == K * N * H * W  # the global count


def test_ring_allreduce_fold_order(orc):
    """src/comm.cpp:288-315: chunk c of the buffer is left-folded in rank order
    c, c+1, ... -- visible with values whose float sum depends on the order"""
    K, n = 3, 7
    bufs = np.zeros((K, n), np.float32)
    bufs[:, :] = np.array([1e8, 1.0, -1e8], np.float32)[:, None]
    orc.orc_ring_allreduce_sum(p(bufs), K, n)
    chunks = [(0, 3), (3, 2), (5, 2)]  # ring_chunks(7, 3)
    for c, (at, ln) in enumerate(chunks):
        vals = [np.float32([1e8, 1.0, -1e8][(c + j) % K]) for j in range(K)]
        acc = vals[0]
        for v in vals[1:]:
            acc = np.float32(acc + v)
        assert np.all(bufs[:, at:at + ln] == acc)
    assert not np.all(bufs[:, 0] == bufs[:, 5])  # the order is observable (0 vs 1)
