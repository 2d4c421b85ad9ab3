"""Run the C4 training step a few times (eager first step, then the CUDA graph)
and bracket exactly ONE graph step with cudaProfilerStart/Stop, for
    ncu --profile-from-start off ... python tools/one_step.py [c4] [warm steps]
(the launch list of one step: profiles/r01_launches_*.csv)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_05831_b200 import detector as D  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    p = D.preset(cfg)
    det = D.Detector(p, device=0)
    B = p.batch
    imgs = torch.zeros((B, p.img_h, p.img_w, 8), dtype=torch.float16, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(1234)
    imgs[..., :3] = torch.randn((B, p.img_h, p.img_w, 3), generator=g, device="cuda", dtype=torch.float16)
    # the profiled step: after `warm` steps (the RoI distribution -- and with
    # it the RoIAlign backward's cost -- settles after the first ~15 steps)
    warm = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    for i in range(warm):
        det.feed(D.batch_slots(i + 1, 0, 1, B), images=imgs, images_on_host=False)
        det.step()
    torch.cuda.synchronize()
    det.feed(D.batch_slots(warm + 1, 0, 1, B), images=imgs, images_on_host=False)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    det.step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("kernels per step (graph):", det.kernel_launches())
    det.close()


if __name__ == "__main__":
    main()
