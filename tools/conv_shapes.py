"""Representative conv launches for an ncu --set full capture (one launch each
after a warm-up): the res5 3x3 fprop (the FLOP-dominant RoI-head shape), the
res4 3x3 fprop (small-M backbone GEMM) and the res2 1x1 64->256 fprop (thin,
HBM-bound backbone layer), all through the C ABI (sdb_conv_fprop)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_05831_b200 import simdet as sd  # noqa: E402

SHAPES = [  # (N, H, W, C, K, R, stride)
    (1024, 7, 7, 512, 512, 3, 1),
    (2, 50, 84, 256, 256, 3, 1),
    (2, 200, 334, 64, 256, 1, 1),
]
if len(sys.argv) > 1 and sys.argv[1] == "res5_1x1":
    SHAPES = [(1024, 7, 7, 512, 2048, 1, 1), (1024, 7, 7, 2048, 512, 1, 1)]
g = torch.Generator(device="cuda").manual_seed(0)
ops = []
for (N, H, W, C, K, R, s) in SHAPES:
    x = torch.randn((N, H, W, C), generator=g, device="cuda").half()
    w = (torch.randn((K, R, R, C), generator=g, device="cuda") * 0.05).half()
    ops.append((x, w, s, R // 2))
for x, w, s, p in ops:  # warm-up (tensor maps, function attributes)
    sd.conv_fprop_nhwc(x, w, s, p)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for x, w, s, p in ops:
    sd.conv_fprop_nhwc(x, w, s, p)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
