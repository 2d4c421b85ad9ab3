"""Per-step GPU times (CUDA events) and host issue times of back-to-back steps (diagnostic)."""
import sys, time
sys.path.insert(0, ".")
import torch, ctypes as C
from paper_1903_05831_b200 import detector as D
p = D.preset(sys.argv[1] if len(sys.argv) > 1 else "c5")
det = D.Detector(p)
lb = D.L(); lb.sdb_ctx_stream.restype = C.c_void_p
stream = torch.cuda.ExternalStream(lb.sdb_ctx_stream(det.ctx))
B = p.batch
imgs = torch.zeros((4, B, p.img_h, p.img_w, 8), dtype=torch.float16, device="cuda")
imgs[..., :3] = torch.randn((4, B, p.img_h, p.img_w, 3), device="cuda").half()
torch.cuda.synchronize()
n = 0
def one(i):
    global n
    n += 1
    det.feed(D.batch_slots(n, 0, 1, B), images=imgs[i % 4], images_on_host=False)
    det.step()
for i in range(5): one(i)
det.losses(); torch.cuda.synchronize()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(31)]
t0 = time.time()
evs[0].record(stream)
hs = []
for i in range(30):
    h0 = time.time(); one(i); hs.append(time.time() - h0)
    evs[i + 1].record(stream)
torch.cuda.synchronize()
print("host per step ms", [round(h * 1e3, 2) for h in hs])
print("gpu per step ms", [round(evs[i].elapsed_time(evs[i + 1]), 2) for i in range(30)])
print("losses", det.losses())
