"""TEST INFRASTRUCTURE ONLY -- an independent checker for the Faster R-CNN C4
training step at sizes the CPU oracle cannot reach (BASELINE config C4:
R50-C4, 800x1333, 512 RoIs/img).

The same graph as oracle/detector_ref.cpp (the reference Tape restatement:
stem 7x7/2 -> max-pool -> res2..res4 bottlenecks, stride in the 1x1 ->
RPN 3x3 + ReLU, 1x1 cls / bbox -> RoIAlign (aligned, sampling ratio 2) ->
res5 -> average pool -> fc cls / fc bbox; losses RPN sigmoid BCE, RPN
smooth-L1 (beta 1/9, / rpn_batch * images), softmax CE (src/model.cpp:101-151),
RCNN class-specific smooth-L1 (beta 1, / #RoIs)), written with torch ops and
torch autograd, teacher-forced on the discrete decisions the GPU step made
(anchor labels/targets, sampled RoIs/labels/targets) -- which the parity tests
check separately, bit for bit, against the restatement.

  mode 0  BN + ReLU (config C1)
  mode 2  InPlace-ABN graph in fp32 (the C2/C4 network without fp16 rounding)
  mode 1  the reference's fp16 contract emulated: every
          op output rounded RNE to binary16 (src/tensor.cpp:59-82), every
          node's incoming gradient rounded to binary16 (src/autograd.cpp:439),
          conv/fc weights used as fp16 shadows (src/trainer.cpp:222-227) and
          their gradients finalised in fp16 (src/autograd.cpp:481); BN
          statistics in fp64 (src/syncbn.cpp:29-39, src/memopt.cpp:247-259).

Nothing here is the product: libsdb never imports it.  It is pinned against
the reference-Tape oracle at small sizes by tests/test_torch_checker_cpu.py.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F


class _Q(torch.autograd.Function):
    """binary16 RNE rounding of a value AND of the gradient flowing into it"""

    @staticmethod
    def forward(ctx, x):
        return x.half().float()

    @staticmethod
    def backward(ctx, g):
        return g.half().float()


def _stage_cfg(blocks):
    return [("res2", blocks[0], 64, 256, 1), ("res3", blocks[1], 128, 512, 2), ("res4", blocks[2], 256, 1024, 2)]


class TorchDetector:
    """One forward/backward of the detector with torch autograd.

    params: {name: np.ndarray} in the reference layouts (conv OIHW, fc [in,out],
    BN [C]) -- the fp32 masters as sdb_det_get_param returns them."""

    def __init__(self, params: dict, mode: int, blocks, A: int, pool: int, device="cpu", eps=1e-5, slope=0.1,
                 sampling_ratio=2, rpn_batch=256, dtype=torch.float32):
        """dtype=torch.float64 (modes 0/2) runs the same graph in double: the
        fp32 arithmetic noise floor of each gradient tensor (its conditioning)"""
        self.mode, self.blocks, self.A, self.pool = mode, tuple(blocks), A, pool
        self.eps, self.slope, self.sr, self.rpn_batch = eps, slope, sampling_ratio, rpn_batch
        self.dev = torch.device(device)
        self.dt = dtype if mode != 1 else torch.float32
        self.p = {}
        for k, v in params.items():
            t = torch.from_numpy(np.ascontiguousarray(v, np.float32)).to(self.dev, self.dt)
            if mode == 1 and not (k.endswith(".gamma") or k.endswith(".beta")):
                t = t.half().float()  # fp16 shadow of the master
            self.p[k] = t.requires_grad_(True)

    # -------------------------------------------------------------- ops
    def q(self, x):
        return _Q.apply(x) if self.mode == 1 else x

    def conv(self, x, name, stride, pad):
        return self.q(F.conv2d(x, self.p[name], stride=stride, padding=pad))

    def norm(self, x, name, act: bool, identity: bool):
        g, b = self.p[name + ".gamma"], self.p[name + ".beta"]
        xd = x.double()
        mean = xd.mean(dim=(0, 2, 3))
        var = torch.clamp((xd * xd).mean(dim=(0, 2, 3)) - mean * mean, min=0.0)
        invstd = (1.0 / torch.sqrt(var + self.eps)).to(self.dt)
        y = g.view(1, -1, 1, 1) * (x - mean.to(self.dt).view(1, -1, 1, 1)) * invstd.view(1, -1, 1, 1) + b.view(1, -1, 1, 1)
        if self.mode == 0:
            y = self.q(y)
            return self.q(F.relu(y)) if act else y
        # InPlace-ABN: leaky(slope) for bn1/bn2/stem, identity (slope 1) for bn3/down
        if not identity:
            y = F.leaky_relu(y, self.slope)
        return self.q(y)

    def act(self, x):
        return self.q(F.relu(x) if self.mode == 0 else F.leaky_relu(x, self.slope))

    def block(self, x, pref, first, stride):
        h = self.conv(x, pref + ".conv1", stride if first else 1, 0)
        h = self.norm(h, pref + ".bn1", True, False)
        h = self.conv(h, pref + ".conv2", 1, 1)
        h = self.norm(h, pref + ".bn2", True, False)
        h = self.conv(h, pref + ".conv3", 1, 0)
        h = self.norm(h, pref + ".bn3", False, True)
        sc = x
        if first:
            sc = self.conv(x, pref + ".down", stride, 0)
            sc = self.norm(sc, pref + ".down_bn", False, True)
        return self.act(self.q(h + sc))

    def stage(self, x, pref, n, stride):
        for b in range(n):
            x = self.block(x, f"{pref}.{b}", b == 0, stride)
        return x

    # -------------------------------------------------------------- step
    def step(self, images, a_labels, a_targets, rois, roi_labels, roi_targets, grad_scale=1.0):
        """images [N,3,H,W] (fp32 values; fp16-valued in mode 1), a_labels int8
        [N, nA], a_targets [N, nA, 4], rois [R,5], roi_labels [R], roi_targets
        [R,4].  Returns (losses[4] float64, grads {name: np.ndarray} scaled by
        grad_scale and finalised in the leaf dtype, rpn logits NCHW)."""
        from torchvision.ops import roi_align
        dev = self.dev
        T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev, self.dt)
        x = T(images)
        if self.mode == 1:
            x = x.half().float()
        N = x.shape[0]
        h = self.conv(x, "stem.conv", 2, 3)
        h = self.norm(h, "stem.bn", True, False)
        h = self.q(F.max_pool2d(h, 3, 2, 1))
        for pref, n, _, _, stride in _stage_cfg(self.blocks):
            h = self.stage(h, pref, n, stride)
        c4 = h
        r = self.q(F.relu(self.conv(c4, "rpn.conv", 1, 1)))
        logits = self.conv(r, "rpn.cls", 1, 0)
        deltas = self.conv(r, "rpn.bbox", 1, 0)
        A = self.A
        lab = torch.as_tensor(np.ascontiguousarray(a_labels)).to(dev).reshape(-1).long()
        lg = logits.permute(0, 2, 3, 1).reshape(-1)
        valid = lab >= 0
        cnt = max(int(valid.sum()), 1)
        l1 = F.binary_cross_entropy_with_logits(lg[valid], lab[valid].to(self.dt), reduction="sum") / cnt
        dl = deltas.permute(0, 2, 3, 1).reshape(-1, 4)
        fg = lab == 1
        beta = 1.0 / 9.0
        d = dl[fg] - T(a_targets).reshape(-1, 4)[fg]
        ad = d.abs()
        l2 = torch.where(ad < beta, 0.5 * d * d / beta, ad - 0.5 * beta).sum() / float(self.rpn_batch * N)
        # RoI head
        rois_t = T(rois)
        f = self.q(roi_align(c4, rois_t, output_size=self.pool, spatial_scale=1.0 / 16.0, sampling_ratio=self.sr,
                             aligned=True))
        self.roi_feat = f
        if self.blocks[3] > 0:
            f = self.stage(f, "res5", self.blocks[3], 2)
        pooled = self.q(f.mean(dim=(2, 3)))
        cls = self.q(pooled @ self.p["fc.cls"])
        box = self.q(pooled @ self.p["fc.bbox"])
        self.inter = {"c4": c4.detach(), "roi_feat": self.roi_feat.detach(), "head_out": f.detach(),
                      "pooled": pooled.detach(), "cls": cls.detach(), "box": box.detach()}
        rl = torch.as_tensor(np.ascontiguousarray(roi_labels)).to(dev).long()
        rv = rl >= 0
        l3 = F.cross_entropy(cls[rv], rl[rv], reduction="mean")
        # the reported value follows the reference CE op (src/model.cpp:117-134):
        # probabilities stashed as float, loss = mean(-log(max(1e-30, p_y))) --
        # a row whose p_y underflows float contributes 69.08, not its true
        # -log p_y (logits reach ~100 at C4); the backward is (p - onehot) as here
        with torch.no_grad():
            p_y = torch.softmax(cls[rv].double(), 1).float().gather(1, rl[rv][:, None]).squeeze(1).double()
            l3_value = (-torch.log(torch.clamp(p_y, min=1e-30))).mean()
        R = int(rv.sum())
        rfg = (rl > 0).nonzero().squeeze(1)
        sel = box[rfg.unsqueeze(1), (4 * rl[rfg]).unsqueeze(1) + torch.arange(4, device=dev)]
        d = sel - T(roi_targets)[rfg]
        ad = d.abs()
        l4 = torch.where(ad < 1.0, 0.5 * d * d, ad - 0.5).sum() / float(R)
        total = l1 + l2 + l3 + l4
        (total * grad_scale).backward()
        grads = {}
        for k, v in self.p.items():
            g = v.grad if v.grad is not None else torch.zeros_like(v)
            if self.mode == 1 and not (k.endswith(".gamma") or k.endswith(".beta")):
                g = g.half().float()  # leaf dtype F16 (src/autograd.cpp:481)
            grads[k] = g.detach().float().cpu().numpy()
        losses = np.array([float(v.detach()) for v in (l1, l2, l3_value, l4)], np.float64)
        return losses, grads, logits.detach().float().cpu().numpy()


def gpu_params(det) -> dict:
    """{name: fp32 master (reference layout)} of a libsdb detector"""
    return {det.params[i][0]: det.get_param(i) for i in range(det.n_tensors)}


def run_checker(det, params, s, mode, grad_scale, device, dtype=torch.float32, inter=None):
    """teacher-forced TorchDetector step on the GPU step's decisions `s`
    (tests.det_parity.gpu_state); returns (losses, flat grads in pack order, logits);
    `inter` (a dict) receives the forward intermediates (c4, roi_feat, head_out,
    pooled, cls, box) as numpy arrays"""
    pr = det.p
    img = np.ascontiguousarray(s["images"][..., :3].astype(np.float32).transpose(0, 3, 1, 2))
    td = TorchDetector(params, mode, pr.blocks, det.A, pr.pool, device=device, dtype=dtype)
    losses, grads, lg = td.step(img, s["a_labels"], s["a_targets"], s["rois"], s["roi_labels"], s["roi_targets"],
                                grad_scale)
    flat = np.concatenate([grads[det.params[i][0]].ravel() for i in range(det.n_tensors)]).astype(np.float32)
    if inter is not None:
        inter.update({k: v.float().cpu().numpy() for k, v in td.inter.items()})
    return losses, flat, lg
