"""Host-side wrapper of the libsdb Faster R-CNN C4 training step (C ABI
``sdb_det_*``).  The step itself -- forward, target assignment, losses,
backward, bucketed NCCL allreduce, loss-scaled fused SGD -- is the C++ driver
in csrc/detector.cpp; this module only builds configs, feeds synthetic batches
and reads results.  Mirrors the reference's run_training step contract
(src/trainer.cpp:217-271): global-batch slots (step-1)*K*b + rank*b + j
(src/dataset.cpp:94) key both the images and the RPN/RCNN sampling RNG.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import check, lib

_P, _I, _L, _D = C.c_void_p, C.c_int, C.c_int64, C.c_double


class DetConfig(C.Structure):
    _fields_ = [
        ("mode", C.c_int), ("batch", C.c_int), ("img_h", C.c_int), ("img_w", C.c_int),
        ("blocks", C.c_int * 4), ("num_classes", C.c_int), ("rpn_channels", C.c_int),
        ("n_scales", C.c_int), ("n_ratios", C.c_int), ("scales", C.c_float * 8), ("ratios", C.c_float * 8),
        ("pre_nms", C.c_int), ("post_nms", C.c_int), ("nms_iou", C.c_double),
        ("rpn_batch", C.c_int), ("rpn_fg_frac", C.c_double), ("rpn_fg_thr", C.c_double), ("rpn_bg_thr", C.c_double),
        ("roi_batch", C.c_int), ("roi_fg_frac", C.c_double), ("roi_fg_thr", C.c_double), ("roi_bg_hi", C.c_double),
        ("roi_bg_lo", C.c_double), ("pool", C.c_int), ("sampling_ratio", C.c_int),
        ("lr", C.c_float), ("momentum", C.c_float), ("eps", C.c_float), ("slope", C.c_float),
        ("dynamic_scale", C.c_int), ("scale_init", C.c_double), ("growth_interval", C.c_int64),
        ("growth", C.c_double), ("backoff", C.c_double), ("min_scale", C.c_double), ("max_scale", C.c_double),
        ("seed", C.c_uint64), ("max_gt", C.c_int), ("bucket_mb", C.c_double), ("shard_optimizer", C.c_int),
        ("sync_bn", C.c_int), ("checkpoint", C.c_int),
    ]


@dataclass
class Preset:
    """A BASELINE.json configuration (configs[0..4])."""
    name: str
    mode: int
    batch: int
    img_h: int
    img_w: int
    blocks: tuple
    num_classes: int
    scales: tuple
    ratios: tuple = (0.5, 1.0, 2.0)
    pre_nms: int = 2000
    post_nms: int = 300
    roi_batch: int = 128
    pool: int = 7
    gt_mode: str = "fixed8"    # fixed8 | poisson7
    gt_wh: tuple = (16.0, 128.0)
    dynamic_scale: int = 0
    scale_init: float = 128.0
    growth_interval: int = 1000
    lr: float = 0.01
    momentum: float = 0.9
    seed: int = 0
    max_gt: int = 32
    extra: dict = field(default_factory=dict)

    def to_c(self) -> DetConfig:
        c = DetConfig()
        c.mode, c.batch, c.img_h, c.img_w = self.mode, self.batch, self.img_h, self.img_w
        for i, b in enumerate(self.blocks):
            c.blocks[i] = b
        c.num_classes, c.rpn_channels = self.num_classes, 512
        c.n_scales, c.n_ratios = len(self.scales), len(self.ratios)
        for i, s in enumerate(self.scales):
            c.scales[i] = s
        for i, r in enumerate(self.ratios):
            c.ratios[i] = r
        c.pre_nms, c.post_nms, c.nms_iou = self.pre_nms, self.post_nms, 0.7
        c.rpn_batch, c.rpn_fg_frac, c.rpn_fg_thr, c.rpn_bg_thr = 256, 0.5, 0.7, 0.3
        c.roi_batch, c.roi_fg_frac, c.roi_fg_thr, c.roi_bg_hi, c.roi_bg_lo = self.roi_batch, 0.25, 0.5, 0.5, 0.0
        c.pool, c.sampling_ratio = self.pool, 2
        c.lr, c.momentum, c.eps, c.slope = self.lr, self.momentum, 1e-5, 0.1
        c.dynamic_scale, c.scale_init, c.growth_interval = self.dynamic_scale, self.scale_init, self.growth_interval
        c.growth, c.backoff, c.min_scale, c.max_scale = 2.0, 0.5, 1.0, 16777216.0
        c.seed, c.max_gt, c.bucket_mb = self.seed, self.max_gt, 25.0
        c.shard_optimizer = 1
        for k, v in self.extra.items():
            setattr(c, k, v)
        return c


def preset(name: str, **kw) -> Preset:
    """BASELINE.json configs: c1 tiny fp32 / c2 tiny fp16+IABN / c4 R50-C4 b2 / c5 R50-C4 b4."""
    tiny = dict(img_h=256, img_w=256, blocks=(1, 1, 1, 0), num_classes=10, scales=(32.0, 64.0, 128.0),
                pre_nms=2000, post_nms=300, roi_batch=128, pool=7, gt_mode="fixed8", gt_wh=(16.0, 128.0))
    r50 = dict(img_h=800, img_w=1333, blocks=(3, 4, 6, 3), num_classes=80,
               scales=(32.0, 64.0, 128.0, 256.0, 512.0), pre_nms=12000, post_nms=2000, roi_batch=512, pool=14,
               gt_mode="poisson7", gt_wh=(8.0, 512.0))
    table = {
        "c1": dict(tiny, mode=0, batch=2, scale_init=1.0),
        "c2": dict(tiny, mode=1, batch=2, scale_init=128.0),
        "c4": dict(r50, mode=1, batch=2, scale_init=128.0),
        "c5": dict(r50, mode=1, batch=4, dynamic_scale=1, scale_init=32768.0, growth_interval=1000),
    }
    d = dict(table[name])
    d.update(kw)
    return Preset(name=name, **d)


_SIGS = {
    "sdb_det_create": [_P, C.POINTER(DetConfig), C.POINTER(_P)],
    "sdb_det_destroy": [_P],
    "sdb_det_num_params": [_P, C.POINTER(_I), C.POINTER(_L), C.POINTER(_L)],
    "sdb_det_param_info": [_P, _I, C.c_char_p, _I, C.POINTER(_L), C.POINTER(_I), C.POINTER(_I)],
    "sdb_det_get_param": [_P, _I, _P],
    "sdb_det_set_param": [_P, _I, _P],
    "sdb_det_get_grad": [_P, _I, _P],
    "sdb_det_get_velocity": [_P, _I, _P],
    "sdb_det_save_checkpoint": [_P, C.c_char_p, C.c_uint64, _L],
    "sdb_det_load_checkpoint": [_P, C.c_char_p, _P, _P],
    "sdb_det_set_velocity": [_P, _I, _P],
    "sdb_det_set_batch": [_P, _P, _I, _P, _P, _P, _P],
    "sdb_det_synth_images": [_P, _P],
    "sdb_det_step": [_P],
    "sdb_det_read_losses": [_P, _P, C.POINTER(_D), C.POINTER(_I)],
    "sdb_det_train_step_host": [_P, _P, _P, _P, _P, _P, _P],
    "sdb_det_train_step_host_nchw": [_P, _P, _P, _P, _P, _P, _P],
    "sdb_det_export": [_P, _I, _P, _L, C.POINTER(_L)],
    "sdb_det_dims": [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)],
    "sdb_det_kernel_launches": [_P, C.POINTER(_L)],
    "sdb_det_memory": [_P, C.POINTER(_L), C.POINTER(_L), C.POINTER(_I)],
    "sdb_det_profile": [_P, _P, _P, _P, _P, _I],
    "sdb_det_profile_record": [_P, _I, C.POINTER(_I), C.c_char_p, _I, C.POINTER(_D), C.POINTER(_D), C.POINTER(_D)],
    "sdb_ctx_create": [_I, _I, _I, _P, C.POINTER(_P)],
    "sdb_ctx_destroy": [_P],
    "sdb_get_nccl_unique_id": [_P],
}
_done = False


def L():
    global _done
    lb = lib()
    if not _done:
        for n, a in _SIGS.items():
            f = getattr(lb, n)
            f.argtypes = a
            f.restype = C.c_int
        _done = True
    return lb


def make_gt(p: Preset, slot: int):
    """Synthetic ground truth for one image (host 'data loader'): centres
    uniform over the image, w/h log-uniform in gt_wh, clipped; classes 1..C."""
    rng = np.random.default_rng([p.seed, 0x9d7, slot])
    n = 8 if p.gt_mode == "fixed8" else max(1, int(rng.poisson(7)))
    n = min(n, p.max_gt)
    cx = rng.uniform(0, p.img_w, n)
    cy = rng.uniform(0, p.img_h, n)
    lo, hi = np.log(p.gt_wh[0]), np.log(p.gt_wh[1])
    w = np.exp(rng.uniform(lo, hi, n))
    h = np.exp(rng.uniform(lo, hi, n))
    boxes = np.stack([np.clip(cx - w / 2, 0, p.img_w), np.clip(cy - h / 2, 0, p.img_h),
                      np.clip(cx + w / 2, 0, p.img_w), np.clip(cy + h / 2, 0, p.img_h)], 1).astype(np.float32)
    cls = rng.integers(1, p.num_classes + 1, n).astype(np.int32)
    return boxes, cls


def batch_slots(step: int, rank: int, world: int, b: int):
    """global batch slots of src/dataset.cpp:94 (1-based step)"""
    return np.array([(step - 1) * world * b + rank * b + j for j in range(b)], np.int64)


class Detector:
    def __init__(self, p: Preset, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 force_comm: bool = False):
        """force_comm (world 1 only): build a 1-rank NCCL communicator so the
        data-parallel code path -- bucket allreduces inside the captured step,
        the loss and BN-gradient allreduces -- runs on one GPU."""
        self.p = p
        lb = L()
        if force_comm and nccl_id is None:
            if world != 1:
                raise ValueError("force_comm is for world == 1; pass the shared nccl_id at world > 1")
            buf = C.create_string_buffer(128)
            check(lb.sdb_get_nccl_unique_id(buf))
            nccl_id = bytes(buf.raw)
        self.ctx = _P()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        check(lb.sdb_ctx_create(device, rank, world, idbuf, C.byref(self.ctx)))
        self.cfg = p.to_c()
        self.h = _P()
        check(lb.sdb_det_create(self.ctx, C.byref(self.cfg), C.byref(self.h)))
        self.rank, self.world = rank, world
        nt, nw, nb = _I(), _L(), _L()
        check(lb.sdb_det_num_params(self.h, C.byref(nt), C.byref(nw), C.byref(nb)))
        self.n_tensors, self.n_w, self.n_bn = nt.value, nw.value, nb.value
        fh, fw, A, Ap = _I(), _I(), _I(), _I()
        check(lb.sdb_det_dims(self.h, C.byref(fh), C.byref(fw), C.byref(A), C.byref(Ap)))
        self.feat_h, self.feat_w, self.A, self.A_pad = fh.value, fw.value, A.value, Ap.value
        self.params = [self.param_info(i) for i in range(self.n_tensors)]

    def close(self):
        if self.h:
            L().sdb_det_destroy(self.h)
            L().sdb_ctx_destroy(self.ctx)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def param_info(self, i):
        name = C.create_string_buffer(128)
        shape = (_L * 4)()
        nd, kind = _I(), _I()
        check(L().sdb_det_param_info(self.h, i, name, 128, shape, C.byref(nd), C.byref(kind)))
        return name.value.decode(), tuple(shape[: nd.value]), kind.value

    def get_param(self, i) -> np.ndarray:
        _, shape, _ = self.params[i]
        out = np.zeros(shape, np.float32)
        check(L().sdb_det_get_param(self.h, i, out.ctypes.data_as(_P)))
        return out

    def set_param(self, i, v: np.ndarray):
        v = np.ascontiguousarray(v, np.float32)
        check(L().sdb_det_set_param(self.h, i, v.ctypes.data_as(_P)))

    def get_grad(self, i) -> np.ndarray:
        _, shape, _ = self.params[i]
        out = np.zeros(shape, np.float32)
        check(L().sdb_det_get_grad(self.h, i, out.ctypes.data_as(_P)))
        return out

    def get_velocity(self, i) -> np.ndarray:
        _, shape, _ = self.params[i]
        out = np.zeros(shape, np.float32)
        check(L().sdb_det_get_velocity(self.h, i, out.ctypes.data_as(_P)))
        return out

    def gt_batch(self, slots):
        p = self.p
        B = len(slots)
        boxes = np.zeros((B, p.max_gt, 4), np.float32)
        cls = np.zeros((B, p.max_gt), np.int32)
        cnt = np.zeros(B, np.int32)
        for j, s in enumerate(slots):
            b, c = make_gt(p, int(s))
            boxes[j, : len(b)] = b
            cls[j, : len(c)] = c
            cnt[j] = len(b)
        return boxes, cls, cnt

    def feed(self, slots, images=None, images_on_host=True):
        """images: None -> synthesize on device from the slots."""
        slots = np.ascontiguousarray(slots, np.int64)
        boxes, cls, cnt = self.gt_batch(slots)
        self._gt = (boxes, cls, cnt)
        lb = L()
        if images is None:
            check(lb.sdb_det_synth_images(self.h, slots.ctypes.data_as(_P)))
            img_ptr = None
        else:
            img_ptr = _P(images.data_ptr()) if hasattr(images, "data_ptr") else images.ctypes.data_as(_P)
        check(lb.sdb_det_set_batch(self.h, img_ptr, 1 if images_on_host else 0, boxes.ctypes.data_as(_P),
                                   cls.ctypes.data_as(_P), cnt.ctypes.data_as(_P), slots.ctypes.data_as(_P)))

    def step(self):
        check(L().sdb_det_step(self.h))

    def losses(self):
        out = (_D * 5)()
        sc = _D()
        ov = _I()
        check(L().sdb_det_read_losses(self.h, out, C.byref(sc), C.byref(ov)))
        return list(out), sc.value, ov.value

    def train_step_host(self, images_host_ptr, slots, gt):
        boxes, cls, cnt = gt
        out = (_D * 5)()
        slots = np.ascontiguousarray(slots, np.int64)
        check(L().sdb_det_train_step_host(self.h, images_host_ptr, boxes.ctypes.data_as(_P), cls.ctypes.data_as(_P),
                                          cnt.ctypes.data_as(_P), slots.ctypes.data_as(_P), out))
        return list(out)

    def train_step_host_nchw(self, images_host_ptr, slots, gt):
        boxes, cls, cnt = gt
        out = (_D * 5)()
        slots = np.ascontiguousarray(slots, np.int64)
        check(L().sdb_det_train_step_host_nchw(self.h, images_host_ptr, boxes.ctypes.data_as(_P), cls.ctypes.data_as(_P),
                                          cnt.ctypes.data_as(_P), slots.ctypes.data_as(_P), out))
        return list(out)

    def export(self, what: int, dtype=np.uint8) -> np.ndarray:
        n = _L()
        check(L().sdb_det_export(self.h, what, None, 0, C.byref(n)))
        buf = np.zeros(n.value, np.uint8)
        check(L().sdb_det_export(self.h, what, buf.ctypes.data_as(_P), n.value, C.byref(n)))
        return buf.view(dtype)

    PROFILE_CATS = ["conv_fprop", "conv_dgrad", "conv_wgrad", "norm_fwd", "norm_bwd", "elementwise", "pooling",
                    "targets", "proposal", "roialign_fwd", "roialign_bwd", "losses", "optimizer", "comm"]

    def profile(self):
        """one eager CUDA-event-instrumented step: {category: (ms, flops, bytes, launches)}"""
        n = len(self.PROFILE_CATS)
        ms, fl, by = (_D * n)(), (_D * n)(), (_D * n)()
        la = (_L * n)()
        check(L().sdb_det_profile(self.h, ms, fl, by, la, n))
        return {c: (ms[i], fl[i], by[i], la[i]) for i, c in enumerate(self.PROFILE_CATS)}

    def profile_records(self):
        """labelled records of the last profile() step: [(category, label, ms, flops, bytes)]"""
        lb = L()
        n = lb.sdb_det_profile_record(self.h, -1, None, None, 0, None, None, None)
        out = []
        for k in range(n):
            cat, ms, fl, by = _I(), _D(), _D(), _D()
            lab = C.create_string_buffer(160)
            check(lb.sdb_det_profile_record(self.h, k, C.byref(cat), lab, 160, C.byref(ms), C.byref(fl), C.byref(by)))
            out.append((self.PROFILE_CATS[cat.value], lab.value.decode(), ms.value, fl.value, by.value))
        return out

    def save_checkpoint(self, path: str, step: int, config_digest: int = 0):
        """SDCK v1 file (src/checkpoint.cpp:47-84): masters, velocity, loss-scale state"""
        check(L().sdb_det_save_checkpoint(self.h, path.encode(), config_digest, step))

    def load_checkpoint(self, path: str):
        """restores the training state; returns (step, config_digest)"""
        dg, st = C.c_uint64(), _L()
        check(L().sdb_det_load_checkpoint(self.h, path.encode(), C.byref(dg), C.byref(st)))
        return st.value, dg.value

    def memory(self):
        """(backbone activation bytes, device bytes, checkpoint segments)"""
        a, t, sg = _L(), _L(), _I()
        check(L().sdb_det_memory(self.h, C.byref(a), C.byref(t), C.byref(sg)))
        return a.value, t.value, sg.value

    def kernel_launches(self) -> int:
        n = _L()
        check(L().sdb_det_kernel_launches(self.h, C.byref(n)))
        return n.value


def smoke_step():
    """One tiny fp16 training step through the C ABI (used by __graft_entry__.smoke)."""
    d = Detector(preset("c2"))
    d.feed(batch_slots(1, 0, 1, 2))
    d.step()
    losses, scale, ov = d.losses()
    assert all(np.isfinite(losses)) and ov == 0, (losses, ov)
    d.close()
    return losses
