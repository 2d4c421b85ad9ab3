"""Dump the sampled RoIs of C4 training steps (diagnostic): gpurun_out/rois_s{step}.npy"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1903_05831_b200 import detector as D  # noqa: E402

at = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,10,20,30,40,50").split(",")]
det = D.Detector(D.preset("c4"))
for s_ in range(1, max(at) + 1):
    det.feed(D.batch_slots(s_, 0, 1, 2))
    det.step()
    if s_ in at:
        det.losses()
        np.save(f"gpurun_out/rois_s{s_}.npy", det.export(4, np.float32).reshape(-1, 5).copy())
det.close()
