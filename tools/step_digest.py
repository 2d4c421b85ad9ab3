"""Bit-identity check between two builds: run K graph steps of a preset on
fixed synthetic images and print a SHA-256 of the losses, parameters and
velocities after every step, plus the per-step GPU times (CUDA events):
    SDB_LIB=scratch/libsdb_base.so python tools/step_digest.py c4 30
    python tools/step_digest.py c4 30
Equal digest lines = bit-identical training trajectories."""
import hashlib
import os
import sys

import ctypes as C
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_05831_b200 import detector as D  # noqa: E402
from tests import det_parity as dp  # noqa: E402


def main():
    preset = sys.argv[1] if len(sys.argv) > 1 else "c4"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    p = D.preset(preset)
    det = D.Detector(p)
    lb = D.L()
    lb.sdb_ctx_stream.restype = C.c_void_p
    stream = torch.cuda.ExternalStream(lb.sdb_ctx_stream(det.ctx))
    B = p.batch
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    imgs = torch.zeros((2, B, p.img_h, p.img_w, 8), dtype=torch.float16, device="cuda")
    imgs[..., :3] = torch.randn((2, B, p.img_h, p.img_w, 3), generator=g, device="cuda").half()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    h = hashlib.sha256()
    ms = []
    for i in range(steps):
        det.feed(D.batch_slots(i + 1, 0, 1, B), images=imgs[i % 2], images_on_host=False)
        evs[i].record(stream)
        det.step()
        evs[i + 1].record(stream)
        losses, scale, ov = det.losses()
        torch.cuda.synchronize()
        ms.append(evs[i].elapsed_time(evs[i + 1]))
        h.update(np.asarray(losses, dtype=np.float64).tobytes())
        if i == steps - 1 or (i + 1) % 10 == 0:
            h.update(dp.flat_params(det).tobytes())
            h.update(dp.flat_velocity(det).tobytes())
            print("step %d digest %s losses %s" % (i + 1, h.hexdigest()[:16], np.round(losses, 6).tolist()))
    t = np.array(ms[10:]) if steps > 15 else np.array(ms)
    print("gpu ms/step min %.3f p25 %.3f median %.3f" % (t.min(), np.percentile(t, 25), np.median(t)))
    det.close()


if __name__ == "__main__":
    main()
