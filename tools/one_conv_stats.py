"""One fprop with fused norm statistics at the res5 expansion shape (RoI head
1x1 512 -> 2048, 1024 RoIs) after a warm-up, bracketed by cudaProfilerStart/
Stop, for an `ncu --profile-from-start off --set full` capture."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_05831_b200 import simdet as sd  # noqa: E402

N, H, W, C, K = 1024, 7, 7, 512, 2048
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((N, H, W, C), generator=g, device="cuda").half()
w = (torch.randn((K, 1, 1, C), generator=g, device="cuda") * 0.05).half()
for _ in range(3):
    sd.conv_fprop_stats_nhwc(x, w, 1, 0, iabn=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
sd.conv_fprop_stats_nhwc(x, w, 1, 0, iabn=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
