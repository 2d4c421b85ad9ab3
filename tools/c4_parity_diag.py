"""Diagnostic (not a test): per-tensor gradient errors of one C4 step against
the torch checker, with the fp32 noise floor (torch32 vs torch64) and, for the
fp16 graph, the fp16 floor (torch16 vs torch32).  Prints a table."""
import os
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
os.environ["SDB_NO_HEAD_POOL_FUSE"] = "1"  # head_out is exported below (not stored when pooled in place)
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
i32 = {}
l32, g32, _ = run_checker(det, params, s, 2, scale, "cuda", inter=i32)
# forward intermediates: GPU exports vs the fp32 checker
pr = det.p
R = s["rois"].shape[0]
dt = np.float16 if mode == 1 else np.float32
gpu_i = {"c4": det.export(10, dt).reshape(pr.batch, det.feat_h, det.feat_w, 1024).transpose(0, 3, 1, 2),
         "roi_feat": det.export(18, dt).reshape(R, 7, 7, 1024).transpose(0, 3, 1, 2),
         "head_out": det.export(19, dt).reshape(R, 7, 7, 2048).transpose(0, 3, 1, 2),
         "pooled": det.export(20, dt).reshape(R, 2048),
         "cls": det.export(21, dt).reshape(R, -1)[:, :81],
         "box": det.export(22, dt).reshape(R, -1)[:, :324]}
ref_i = dict(i32)
ref_i["roi_feat"] = i32["roi_feat"][:, :, ::2, ::2]
for k in gpu_i:
    a, b = gpu_i[k].astype(np.float32), ref_i[k]
    print("inter %-9s norm-rel %.3e  max-abs %.3e  ref-max %.3e" % (k, norm_rel(a, b), np.abs(a - b).max(), np.abs(b).max()))
rl = s["roi_labels"]
ce_rows = [(i, float(v)) for i, v in enumerate(np.abs(gpu_i["cls"].astype(np.float32) - ref_i["cls"]).max(1))]
ce_rows.sort(key=lambda t: -t[1])
def _ce(lg, lab):
    lg = lg.astype(np.float64)
    m = lg.max(1)
    lse = m + np.log(np.exp(lg - m[:, None]).sum(1))
    return lse - lg[np.arange(lg.shape[0]), lab]
ce_g, ce_r = _ce(gpu_i["cls"], rl), _ce(ref_i["cls"], rl)
print("CE on exported GPU logits %.6f, on checker logits %.6f; largest per-row diffs" % (ce_g.mean(), ce_r.mean()),
      sorted(zip(np.abs(ce_g - ce_r), range(len(rl))))[-5:])
print("worst cls rows:", ce_rows[:8], "labels", [int(rl[i]) for i, _ in ce_rows[:8]])
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
