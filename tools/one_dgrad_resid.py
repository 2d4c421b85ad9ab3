"""One residual dgrad (the RoI head's c1 dgrad: dy [1024,7,7,512] -> dx
[1024,7,7,2048] + addend, leaky mask from a sign bitmap) after a warm-up,
bracketed by cudaProfilerStart/Stop for `ncu --profile-from-start off`."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_05831_b200 import simdet as sd  # noqa: E402

N, H, W, C, K = 1024, 7, 7, 2048, 512
g = torch.Generator(device="cuda").manual_seed(0)
dy = torch.randn((N, H, W, K), generator=g, device="cuda").half()
w = (torch.randn((K, 1, 1, C), generator=g, device="cuda") * 0.05).half()
addend = torch.randn((N, H, W, C), generator=g, device="cuda").half()
y = torch.randn((N, H, W, C), generator=g, device="cuda").half()
bits = sd.sign_bits_nhwc(y)
for _ in range(3):
    sd.conv_dgrad_act_nhwc(dy, w, addend, y, 0.1, 1, 0, y_bits=bits)
torch.cuda.synchronize()
if len(sys.argv) > 1 and sys.argv[1] == "time":
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        sd.conv_dgrad_act_nhwc(dy, w, addend, y, 0.1, 1, 0, y_bits=bits)
    e1.record()
    torch.cuda.synchronize()
    print("residual dgrad 1024x7x7 512->2048: %.1f us" % (e0.elapsed_time(e1) / 20 * 1e3))
    sys.exit(0)
torch.cuda.cudart().cudaProfilerStart()
sd.conv_dgrad_act_nhwc(dy, w, addend, y, 0.1, 1, 0, y_bits=bits)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
