"""RoIAlign microbenchmark on the C4 step's real inputs: runs one C4 training
step, takes its C4 feature map and sampled RoIs (1024 RoIs, 1024 channels,
50x84, P=14 with the res5 stride fold: 7x7 pooled bins), and times
sdb_roialign_fwd_folded / sdb_roialign_bwd_folded with CUDA events (L2 warm,
like inside the step).  Also the C3 shape (P=14, no fold) on the same RoIs.
Prints microseconds and algorithmic GB/s."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1903_05831_b200 import detector as D  # noqa: E402
from paper_1903_05831_b200 import simdet as sd  # noqa: E402

det = D.Detector(D.preset("c4"))
det.feed(D.batch_slots(1, 0, 1, 2))
det.step()
det.losses()
c4 = torch.from_numpy(det.export(10, np.float16).reshape(2, 50, 84, 1024).copy()).cuda()
rois = torch.from_numpy(det.export(4, np.float32).reshape(-1, 5).copy()).cuda()
det.close()
lib = sd.L()
R = rois.shape[0]
for (P, step) in ((14, 2), (14, 1)):
    Po = (P + step - 1) // step
    out = torch.empty((R, Po, Po, 1024), dtype=torch.float16, device="cuda")
    dy = torch.randn((R, Po, Po, 1024), device="cuda").half()
    dx = torch.empty_like(c4)

    def fwd():
        sd.check(lib.sdb_roialign_fwd_folded(sd.ctx(), 1, sd.ptr(c4), 2, 50, 84, 1024, sd.ptr(rois), R, P, 1 / 16, 2, step,
                                             sd.ptr(out), sd.stream()))

    def bwd():
        sd.check(lib.sdb_roialign_bwd_folded(sd.ctx(), 1, sd.ptr(dy), 2, 50, 84, 1024, sd.ptr(rois), R, P, 1 / 16, 2, step,
                                             sd.ptr(dx), sd.stream()))
    for f, name, byts in ((fwd, "fwd", out.numel() * 2 + c4.numel() * 2), (bwd, "bwd", dy.numel() * 2 + dx.numel() * 2)):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        print(f"P={P} step={step} {name}: {us:8.1f} us  {byts / us / 1e3:7.1f} GB/s (algorithmic {byts / 1e6:.1f} MB)")
