"""Interleaved A/B of the C4 graph step: two detectors in one process, one
built with an SDB_* switch set (read at build time), stepped in alternating
blocks so power-cap and clock drift hit both alike:
    python tools/ab_steps.py SDB_NO_POOL_FUSE [preset] [rounds]
prints per-step ms (min / p25 / median) for A (switch unset) and B (set)."""
import os
import sys

import ctypes as C
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_05831_b200 import detector as D  # noqa: E402

switch = sys.argv[1]
preset = sys.argv[2] if len(sys.argv) > 2 else "c4"
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 6
p = D.preset(preset)
B = p.batch
dets = []
for on in (False, True):
    if on:
        os.environ[switch] = "1"
    else:
        os.environ.pop(switch, None)
    dets.append(D.Detector(p))
os.environ.pop(switch, None)
lb = D.L()
lb.sdb_ctx_stream.restype = C.c_void_p
streams = [torch.cuda.ExternalStream(lb.sdb_ctx_stream(d.ctx)) for d in dets]
imgs = torch.zeros((B, p.img_h, p.img_w, 8), dtype=torch.float16, device="cuda")
imgs[..., :3] = torch.randn((B, p.img_h, p.img_w, 3), device="cuda").half()
n = [0, 0]


def block(k, steps):
    d, s = dets[k], streams[k]
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evs[0].record(s)
    for i in range(steps):
        n[k] += 1
        d.feed(D.batch_slots(n[k], 0, 1, B), images=imgs, images_on_host=False)
        d.step()
        evs[i + 1].record(s)
    torch.cuda.synchronize()
    return [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]


for k in (0, 1):
    block(k, 15)  # warm-up: graph capture, RoI distribution settles
t = [[], []]
for r in range(rounds):
    for k in ((0, 1) if r % 2 == 0 else (1, 0)):
        t[k] += block(k, 10)
for k, name in ((0, "A (default)"), (1, "B (%s=1)" % switch)):
    a = np.array(t[k])
    print("%-28s min %.3f  p25 %.3f  median %.3f ms  (%d steps)" % (name, a.min(), np.percentile(a, 25),
                                                                   np.median(a), len(a)))
for d in dets:
    d.close()
