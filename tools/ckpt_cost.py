"""Step time and backbone activation bytes with and without sqrt(L)
checkpointing (diagnostic): python tools/ckpt_cost.py [c4|c5]"""
import sys
import ctypes as C
sys.path.insert(0, ".")
import torch
from paper_1903_05831_b200 import detector as D

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
for ck in (0, 1):
    p = D.preset(name, extra={"checkpoint": ck})
    det = D.Detector(p)
    lb = D.L()
    lb.sdb_ctx_stream.restype = C.c_void_p
    stream = torch.cuda.ExternalStream(lb.sdb_ctx_stream(det.ctx))
    B = p.batch
    imgs = torch.zeros((B, p.img_h, p.img_w, 8), dtype=torch.float16, device="cuda")
    imgs[..., :3] = torch.randn((B, p.img_h, p.img_w, 3), device="cuda").half()
    torch.cuda.synchronize()
    n = 0
    for i in range(15):
        n += 1
        det.feed(D.batch_slots(n, 0, 1, B), images=imgs, images_on_host=False)
        det.step()
    det.losses()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(20):
        n += 1
        det.feed(D.batch_slots(n, 0, 1, B), images=imgs, images_on_host=False)
        det.step()
    e1.record(stream)
    torch.cuda.synchronize()
    act, total, segs = det.memory()
    print(f"{name} checkpoint={ck}: {e0.elapsed_time(e1) / 20:.3f} ms/step, backbone activations "
          f"{act / 2**20:.1f} MiB, device total {total / 2**20:.1f} MiB, segments {segs}", flush=True)
    det.close()
