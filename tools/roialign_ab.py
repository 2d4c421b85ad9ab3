"""RoIAlign timing on FIXED RoI sets (diagnostic A/B between kernel versions):
python tools/roialign_ab.py DIR -- DIR holds rois_s*.npy written by
tools/roi_dump.py (the sampled RoIs of C4 training steps); features and dY are
random (timing does not depend on their values)."""
import glob
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1903_05831_b200 import simdet as sd  # noqa: E402

lib = sd.L()
files = sorted(glob.glob(sys.argv[1] + "/rois_s*.npy"), key=lambda f: int(f.split("_s")[-1][:-4]))
c4 = torch.randn((2, 50, 84, 1024), device="cuda").half()
tot = {}
for fn in files:
    rois = torch.from_numpy(np.load(fn)).cuda()
    R = rois.shape[0]
    line = [fn.split("/")[-1]]
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
        for f, name in ((fwd, "fwd"), (bwd, "bwd")):
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
            line.append(f"P{P}/{step} {name} {us:7.1f}")
    print("  ".join(line), flush=True)
for (P, step, name), v in tot.items():
    print(f"mean: P={P} step={step} {name}: {np.mean(v):8.1f} us (min {min(v):.1f}, max {max(v):.1f})")
