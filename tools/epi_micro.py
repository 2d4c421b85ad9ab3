"""fprop with vs without fused norm statistics (diagnostic): is the statistics
part of the TMA-store epilogue what bounds the 1x1 layers?"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_05831_b200 import simdet as sd  # noqa: E402

SHAPES = [(1024, 7, 7, 512, 2048, 1, 1), (1024, 7, 7, 2048, 512, 1, 1), (2, 200, 334, 64, 256, 1, 1),
          (2, 50, 84, 256, 1024, 1, 1), (2, 100, 167, 128, 512, 1, 1), (2, 50, 84, 256, 256, 3, 1)]
g = torch.Generator(device="cuda").manual_seed(0)
for (N, H, W, C, K, R, s) in SHAPES:
    x = torch.randn((N, H, W, C), generator=g, device="cuda").half()
    w = (torch.randn((K, R, R, C), generator=g, device="cuda") * 0.05).half()
    res = []
    for name, fn in (("plain", lambda: sd.conv_fprop_nhwc(x, w, s, R // 2)),
                     ("stats", lambda: sd.conv_fprop_stats_nhwc(x, w, s, R // 2, iabn=True))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 20 * 1e3)
    fl = 2.0 * N * H * W * C * K * R * R / (s * s)
    print(f"N{N} H{H} W{W} C{C} K{K} R{R}: plain {res[0]:7.1f} us ({fl / res[0] / 1e6:6.0f} TF/s)  "
          f"+stats {res[1]:7.1f} us", flush=True)
