"""How deep the greedy NMS scan goes in the C4 step as training proceeds:
position (in the 12000-candidate top-k order) of the 2000th kept box, per
image, from the step's own RPN outputs through the CPU restatement."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
from oracle import p  # noqa: E402
from paper_1903_05831_b200 import detector as D  # noqa: E402

orc = oracle.orc()
det = D.Detector(D.preset("c4"))
an = det.export(9, np.float32).reshape(-1, 4)
nA = an.shape[0]
A, Ap, fh, fw = det.A, det.A_pad, det.feat_h, det.feat_w
for step in range(1, 61):
    det.feed(D.batch_slots(step, 0, 1, 2))
    det.step()
    if step in (1, 5, 10, 20, 30, 40, 50, 60):
        det.losses()
        lg_all = det.export(7, np.float16).reshape(2, fh * fw, Ap)
        dl_all = det.export(8, np.float16).reshape(2, fh * fw, 4 * Ap)
        depths = []
        for j in range(2):
            lg = np.ascontiguousarray(lg_all[j, :, :A].astype(np.float32).reshape(-1))
            dl = np.ascontiguousarray(dl_all[j, :, :4 * A].astype(np.float32).reshape(-1))
            order = np.zeros(12000, np.int32)
            orc.orc_topk_order(p(lg), nA, 12000, p(order))
            bx = np.zeros((12000, 4), np.float32)
            one = np.ones(4, np.float32)
            orc.orc_decode(p(np.ascontiguousarray(an[order])), p(np.ascontiguousarray(dl.reshape(-1, 4)[order])),
                           12000, p(one), np.float32(np.log(1000 / 16)), 800.0, 1333.0, p(bx))
            keep = np.zeros(2000, np.int32)
            nk = orc.orc_nms_sorted(p(bx), 12000, 0.7, 2000, p(keep))
            depths.append((int(nk), int(keep[nk - 1]) + 1))
        print("step", step, "kept/depth per image", depths, flush=True)
det.close()
