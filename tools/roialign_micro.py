"""RoIAlign microbenchmark on the C4 step's real inputs (diagnostic).

Trains the C4 detector for the given steps and, at each listed step, takes its
C4 feature map and sampled RoIs (1024 RoIs, 1024 channels, 50x84), then times
sdb_roialign_fwd_folded / sdb_roialign_bwd_folded with CUDA events (L2 warm,
like inside the step) for P=14 with the res5 stride fold (7x7 pooled bins, the
step's shape) and without it (14x14, the C3 pooled shape).  The RoI size
distribution -- and with it the backward's cost -- changes as the RPN trains,
so several steps are sampled.  Prints microseconds and algorithmic GB/s.

    python tools/roialign_micro.py [steps,comma,separated] [profile]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1903_05831_b200 import detector as D  # noqa: E402
from paper_1903_05831_b200 import simdet as sd  # noqa: E402

at = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,10,20,30,40,50").split(",")]
prof = len(sys.argv) > 2
det = D.Detector(D.preset("c4"))
samples = []
for s_ in range(1, max(at) + 1):
    det.feed(D.batch_slots(s_, 0, 1, 2))
    det.step()
    if s_ in at:
        det.losses()
        c4 = torch.from_numpy(det.export(10, np.float16).reshape(2, 50, 84, 1024).copy()).cuda()
        rois = torch.from_numpy(det.export(4, np.float32).reshape(-1, 5).copy()).cuda()
        samples.append((s_, c4, rois))
det.close()
lib = sd.L()
tot = {}
for s_, c4, rois in samples:
    R = rois.shape[0]
    w = (rois[:, 3] - rois[:, 1]).clamp(min=0) / 16
    h = (rois[:, 4] - rois[:, 2]).clamp(min=0) / 16
    print(f"step {s_}: RoI size (feature px) mean {float((w * h).sqrt().mean()):.1f}, "
          f"max {float((w * h).sqrt().max()):.1f}", flush=True)
    for (P, step) in ((14, 2), (14, 1)):
        Po = (P + step - 1) // step
        out = torch.empty((R, Po, Po, 1024), dtype=torch.float16, device="cuda")
        dy = torch.randn((R, Po, Po, 1024), device="cuda").half()
        dx = torch.empty_like(c4)

        def fwd():
            sd.check(lib.sdb_roialign_fwd_folded(sd.ctx(), 1, sd.ptr(c4), 2, 50, 84, 1024, sd.ptr(rois), R, P, 1 / 16,
                                                 2, step, sd.ptr(out), sd.stream()))

        def bwd():
            sd.check(lib.sdb_roialign_bwd_folded(sd.ctx(), 1, sd.ptr(dy), 2, 50, 84, 1024, sd.ptr(rois), R, P, 1 / 16,
                                                 2, step, sd.ptr(dx), sd.stream()))
        for f, name, byts in ((fwd, "fwd", out.numel() * 2 + c4.numel() * 2),
                              (bwd, "bwd", dy.numel() * 2 + dx.numel() * 2)):
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
            tot.setdefault((P, step, name), []).append(us)
            print(f"  P={P} step={step} {name}: {us:8.1f} us  {byts / us / 1e3:7.1f} GB/s "
                  f"(algorithmic {byts / 1e6:.1f} MB)", flush=True)
            if prof:  # one more launch inside a profiler window (ncu --profile-from-start off)
                torch.cuda.cudart().cudaProfilerStart()
                f()
                torch.cuda.synchronize()
                torch.cuda.cudart().cudaProfilerStop()
for (P, step, name), v in tot.items():
    print(f"mean over steps {at}: P={P} step={step} {name}: {np.mean(v):8.1f} us (min {min(v):.1f}, max {max(v):.1f})")
