"""Faster R-CNN step parity harness: libsdb (C ABI) vs the oracle.

Per step:
  discrete, BIT-EXACT given the GPU's fp32/fp16 tensors:
    anchors                     == orc_anchors
    anchor labels + targets     == orc_anchor_targets(anchors, GT, key)
    RPN proposals (+count)      == orc_proposals(GPU logits, GPU deltas)
    sampled RoIs/labels/targets == orc_proposal_targets(GPU proposals, GT, key)
  continuous, on the reference Tape (oracle/detector_ref.cpp) fed the GPU's
  decisions (teacher forcing): the four losses, every parameter gradient and
  the per-step parameter deltas (after apply_sgd, src/trainer.cpp:86-94).
"""
import ctypes as C

import numpy as np

import oracle
from oracle import p as ptr

ORC_KEY_RPN = 0xA11C0000
ORC_KEY_RCNN = 0x5A3B0000


def ref_cfg(det):
    pr = det.p
    c = oracle.RefDetCfg()
    c.mode, c.batch, c.img_h, c.img_w = pr.mode, pr.batch, pr.img_h, pr.img_w
    for i, b in enumerate(pr.blocks):
        c.blocks[i] = b
    c.num_classes, c.rpn_channels, c.A = pr.num_classes, 512, det.A
    c.pool, c.sampling_ratio, c.rpn_batch = pr.pool, 2, 256
    c.eps, c.slope = 1e-5, 0.1
    return c


def check_param_order(det, cfg):
    ref = oracle.ref()
    cap = 512
    names = C.create_string_buffer(64 * cap)
    shapes = np.zeros((cap, 4), np.int64)
    kinds = np.zeros(cap, np.int32)
    n = ref.ref_det_param_list(C.byref(cfg), names, ptr(shapes), ptr(kinds), cap)
    assert n == det.n_tensors
    for i in range(n):
        nm = names.raw[64 * i: 64 * i + 64].split(b"\0")[0].decode()
        gname, gshape, gkind = det.params[i]
        assert nm == gname, (i, nm, gname)
        assert tuple(shapes[i][: len(gshape)]) == gshape, (nm, shapes[i], gshape)
        assert kinds[i] == gkind


def flat_params(det):
    return np.concatenate([det.get_param(i).ravel() for i in range(det.n_tensors)]).astype(np.float32)


def flat_velocity(det):
    return np.concatenate([det.get_velocity(i).ravel() for i in range(det.n_tensors)]).astype(np.float32)


def flat_grads(det):
    return np.concatenate([det.get_grad(i).ravel() for i in range(det.n_tensors)]).astype(np.float32)


def split(det, flat):
    out, o = [], 0
    for (_, shape, _) in det.params:
        n = int(np.prod(shape))
        out.append(flat[o:o + n].reshape(shape))
        o += n
    return out


def gpu_state(det):
    pr = det.p
    B = pr.batch
    dt = np.float16 if pr.mode == 1 else np.float32
    fh, fw, A, Ap = det.feat_h, det.feat_w, det.A, det.A_pad
    nA = fh * fw * A
    s = {}
    s["anchors"] = det.export(9, np.float32).reshape(nA, 4)
    s["a_labels"] = det.export(0, np.int8).reshape(B, nA)
    s["a_targets"] = det.export(1, np.float32).reshape(B, nA, 4)
    s["props"] = det.export(2, np.float32).reshape(B, pr.post_nms, 4)
    s["prop_count"] = det.export(3, np.int32)
    s["rois"] = det.export(4, np.float32).reshape(-1, 5)
    s["roi_labels"] = det.export(5, np.int32)
    s["roi_targets"] = det.export(6, np.float32).reshape(-1, 4)
    s["logits"] = det.export(7, dt).reshape(B, fh, fw, Ap)
    s["deltas"] = det.export(8, dt).reshape(B, fh, fw, 4 * Ap)
    s["images"] = det.export(11, dt).reshape(B, pr.img_h, pr.img_w, 8)
    return s


def check_discrete(det, s, slots):
    """bit-exact checks of every discrete decision against the restated oracle."""
    orc = oracle.orc()
    pr = det.p
    B = pr.batch
    fh, fw, A = det.feat_h, det.feat_w, det.A
    nA = fh * fw * A
    scales = np.array(pr.scales, np.float32)
    ratios = np.array(pr.ratios, np.float32)
    an = np.zeros((nA, 4), np.float32)
    orc.orc_anchors(fh, fw, 16.0, ptr(scales), len(scales), ptr(ratios), len(ratios), ptr(an))
    assert np.array_equal(an.view(np.uint32), s["anchors"].view(np.uint32)), "anchors"
    boxes, cls, cnt = det._gt
    report = {}
    for j in range(B):
        G = int(cnt[j])
        gt = np.ascontiguousarray(boxes[j, :G])
        key_rpn = orc.orc_mix64(ORC_KEY_RPN ^ pr.seed, int(slots[j]))
        key_rcnn = orc.orc_mix64(ORC_KEY_RCNN ^ pr.seed, int(slots[j]))
        lab = np.zeros(nA, np.int8)
        tg = np.zeros((nA, 4), np.float32)
        orc.orc_anchor_targets(ptr(an), nA, ptr(gt), G, float(pr.img_h), float(pr.img_w), key_rpn, 0.7, 0.3, 256, 0.5,
                               ptr(lab), ptr(tg))
        assert np.array_equal(lab, s["a_labels"][j]), f"anchor labels img {j}: {np.flatnonzero(lab != s['a_labels'][j])[:10]}"
        np.testing.assert_allclose(tg, s["a_targets"][j], rtol=1e-6, atol=1e-6)
        # proposals from the GPU's own RPN outputs
        lg = np.ascontiguousarray(s["logits"][j][..., :A].astype(np.float32).reshape(-1))
        dl = np.ascontiguousarray(s["deltas"][j].astype(np.float32).reshape(fh * fw, -1)[:, : 4 * A].reshape(-1))
        rois = np.zeros((pr.post_nms, 4), np.float32)
        sc = np.zeros(pr.post_nms, np.float32)
        k = min(pr.pre_nms, nA)
        order = np.zeros(k, np.int32)
        n = orc.orc_proposals(ptr(lg), ptr(dl), ptr(an), nA, float(pr.img_h), float(pr.img_w), pr.pre_nms, 0.7,
                              pr.post_nms, ptr(rois), ptr(sc), ptr(order))
        assert n == s["prop_count"][j], ("proposal count", n, s["prop_count"][j])
        assert np.array_equal(rois[:n].view(np.uint32), s["props"][j][:n].view(np.uint32)), f"proposals img {j}"
        # sampled RoIs
        Rb = pr.roi_batch
        orois = np.zeros((Rb, 4), np.float32)
        olab = np.zeros(Rb, np.int32)
        otg = np.zeros((Rb, 4), np.float32)
        gcls = np.ascontiguousarray(cls[j, :G])
        S = orc.orc_proposal_targets(ptr(np.ascontiguousarray(rois[:n])), n, ptr(gt), ptr(gcls), G, key_rcnn, 0.5, 0.5,
                                     0.0, Rb, 0.25, ptr(orois), ptr(olab), ptr(otg), None)
        gr = s["rois"][j * Rb:(j + 1) * Rb]
        assert S == int((s["roi_labels"][j * Rb:(j + 1) * Rb] >= 0).sum()), "sampled count"
        assert np.all(gr[:S, 0] == j)
        assert np.array_equal(orois[:S].view(np.uint32), gr[:S, 1:].view(np.uint32)), f"sampled rois img {j}"
        assert np.array_equal(olab[:S], s["roi_labels"][j * Rb: j * Rb + S]), f"roi labels img {j}"
        np.testing.assert_allclose(otg[:S], s["roi_targets"][j * Rb: j * Rb + S], rtol=1e-5, atol=1e-5)
        report[j] = dict(fg_anchors=int((lab == 1).sum()), proposals=int(n), rois=int(S), fg_rois=int((olab > 0).sum()))
    return report


def oracle_step(det, cfg, w_flat, s, grad_scale):
    pr = det.p
    B = pr.batch
    img = np.ascontiguousarray(s["images"][..., :3].astype(np.float32).transpose(0, 3, 1, 2))
    R = s["rois"].shape[0]
    assert (s["roi_labels"] >= 0).all(), "padded RoIs present; oracle expects full batches"
    losses = np.zeros(4, np.float64)
    grads = np.zeros_like(w_flat)
    fh, fw, A = det.feat_h, det.feat_w, det.A
    lg = np.zeros((B, A, fh, fw), np.float32)
    dl = np.zeros((B, 4 * A, fh, fw), np.float32)
    rc = oracle.ref().ref_det_step(C.byref(cfg), ptr(w_flat), ptr(img), ptr(np.ascontiguousarray(s["a_labels"])),
                                   ptr(np.ascontiguousarray(s["a_targets"])), ptr(np.ascontiguousarray(s["rois"])),
                                   ptr(np.ascontiguousarray(s["roi_labels"])),
                                   ptr(np.ascontiguousarray(s["roi_targets"])), R, grad_scale, ptr(losses), ptr(grads),
                                   ptr(lg), ptr(dl))
    assert rc == 0
    return losses, grads, lg, dl
