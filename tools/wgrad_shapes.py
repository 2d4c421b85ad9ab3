"""Backbone wgrad launches for an ncu capture (one launch each after a
warm-up): res4 1x1 256->1024, res4 3x3 256->256, res3 3x3 128->128, through
the C ABI (sdb_conv_wgrad: split-K TMA GEMM + reduce)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_05831_b200 import simdet as sd  # noqa: E402

SHAPES = [  # (N, H, W, C, K, R, stride)
    (2, 50, 84, 256, 1024, 1, 1),
    (2, 50, 84, 256, 256, 3, 1),
    (2, 100, 167, 128, 128, 3, 1),
]
g = torch.Generator(device="cuda").manual_seed(0)
ops = []
for (N, H, W, C, K, R, s) in SHAPES:
    x = torch.randn((N, H, W, C), generator=g, device="cuda").half()
    dy = torch.randn((N, H, W, K), generator=g, device="cuda").half()
    ops.append((x, dy, (K, R, R, C), s, R // 2))
for x, dy, ws, s, p in ops:
    sd.conv_wgrad_nhwc(x, dy, ws, s, p)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * len(ops))]
for i, (x, dy, ws, s, p) in enumerate(ops):
    ev[2 * i].record()
    for _ in range(20):
        sd.conv_wgrad_nhwc(x, dy, ws, s, p)
    ev[2 * i + 1].record()
torch.cuda.synchronize()
for i, (x, dy, ws, s, p) in enumerate(ops):
    N, H, W, C = x.shape
    fl = 2.0 * N * H * W * C * ws[0] * ws[1] * ws[2]
    t = ev[2 * i].elapsed_time(ev[2 * i + 1]) / 20
    print(f"wgrad N{N} H{H} W{W} C{C} K{ws[0]} R{ws[1]}: {t * 1e3:.1f} us  {fl / t / 1e9:.0f} TF/s", flush=True)
torch.cuda.cudart().cudaProfilerStart()
for x, dy, ws, s, p in ops:
    sd.conv_wgrad_nhwc(x, dy, ws, s, p)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
