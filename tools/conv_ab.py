"""Time single conv launches (fprop / dgrad / wgrad through the C ABI) with CUDA
events, L2 left warm (backbone feature maps are L2-resident in the step):
    python tools/conv_ab.py            # the backbone 3x3 shapes
Run twice with and without an SDB_* switch for an A/B."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_05831_b200 import simdet as sd  # noqa: E402

SHAPES = [  # (N, H, W, C, K, R, stride)
    (1024, 7, 7, 512, 2048, 1, 1),
    (1024, 7, 7, 2048, 512, 1, 1),
    (2, 200, 334, 64, 256, 1, 1),
    (2, 50, 84, 256, 256, 3, 1),
    (2, 100, 167, 128, 128, 3, 1),
    (2, 200, 334, 64, 64, 3, 1),
    (2, 50, 84, 1024, 256, 1, 1),
    (2, 50, 84, 256, 1024, 1, 1),
    (2, 100, 167, 512, 128, 1, 1),
    (2, 100, 167, 128, 512, 1, 1),
]


def timeit(fn, n=20, reps=5):
    """per-launch device time of fn, captured n times in one CUDA graph (no host
    launch overhead in the measurement)"""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(n):
            fn()
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(reps):
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / n)
    return best


g = torch.Generator(device="cuda").manual_seed(0)
for (N, H, W, C, K, R, s) in SHAPES:
    x = torch.randn((N, H, W, C), generator=g, device="cuda").half()
    w = (torch.randn((K, R, R, C), generator=g, device="cuda") * 0.05).half()
    y = sd.conv_fprop_nhwc(x, w, s, R // 2)
    dy = torch.randn_like(y)
    flop = 2.0 * y.numel() * C * R * R
    tf = timeit(lambda: sd.conv_fprop_nhwc(x, w, s, R // 2))
    ts = timeit(lambda: sd.conv_fprop_stats_nhwc(x, w, s, R // 2, iabn=True))
    td = timeit(lambda: sd.conv_dgrad_nhwc(dy, w, x.shape, s, R // 2))
    tw = timeit(lambda: sd.conv_wgrad_nhwc(x, dy, w.shape, s, R // 2))
    print(f"N{N} H{H} W{W} C{C} K{K} R{R}: fprop {tf:6.1f} us ({flop / tf / 1e6:5.0f} TF/s)  +stats {ts:6.1f}  "
          f"dgrad {td:6.1f} us ({flop / td / 1e6:5.0f})  wgrad {tw:6.1f} us ({flop / tw / 1e6:5.0f})")
