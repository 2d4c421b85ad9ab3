"""Diagnostic (not a test): per-tensor gradient errors of one C4 step against
the torch checker, with the fp32 noise floor (torch32 vs torch64) and, for the
fp16 graph, the fp16 floor (torch16 vs torch32).  Prints a table."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1903_05831_b200 import detector as D  # noqa: E402
from tests import det_parity as dp  # noqa: E402
from tests.torch_detector import gpu_params, run_checker  # noqa: E402
from tests.util import norm_rel  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 2
at_step = int(sys.argv[2]) if len(sys.argv) > 2 else 1
det = D.Detector(D.preset("c4", mode=mode, scale_init=1.0 if mode != 1 else 128.0))
for st in range(1, at_step):
    det.feed(D.batch_slots(st, 0, 1, det.p.batch))
    det.step()
    print("step", st, det.losses())
params = gpu_params(det)
slots = D.batch_slots(at_step, 0, 1, det.p.batch)
det.feed(slots)
det.step()
losses, scale, ov = det.losses()
s = dp.gpu_state(det)
g = dp.flat_grads(det)
l32, g32, _ = run_checker(det, params, s, 2, scale, "cuda")
torch.cuda.empty_cache()
l64, g64, _ = run_checker(det, params, s, 2, scale, "cuda", dtype=torch.float64)
torch.cuda.empty_cache()
cols = [("gpu-t32", g, g32), ("t32-t64", g32, g64), ("gpu-t64", g, g64)]
if mode == 1:
    l16, g16, _ = run_checker(det, params, s, 1, scale, "cuda")
    cols = [("gpu-t16", g, g16), ("t16-t32", g16, g32)] + cols
print("losses gpu", losses[:4], "t32", l32, "t64", l64, "t16", l16 if mode == 1 else None)
print("rois/labels: fg", int((s["roi_labels"] > 0).sum()), "bg", int((s["roi_labels"] == 0).sum()))
print("%-24s" % "global" + "".join(" %s %.2e" % (n, norm_rel(a, b)) for n, a, b in cols))
sp = {n: (dp.split(det, a), dp.split(det, b)) for n, a, b in cols}
for i, (name, _, _) in enumerate(det.params):
    print("%-24s" % name + "".join(" %s %.2e" % (n, norm_rel(sp[n][0][i], sp[n][1][i])) for n, _, _ in cols))
