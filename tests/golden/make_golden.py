"""Generate tests/golden/reference_golden.npz from the COMPILED REFERENCE
(oracle/_ref/libsimdet_ref.so, built from /root/reference/proj/src).  Run in
the build container (needs the reference); the fixture is committed so the CPU
suite can pin the restated oracle without the reference present.

    python tests/golden/make_golden.py
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import p  # noqa: E402


def main():
    ref = oracle.ref()
    rng = np.random.default_rng(2026)
    out = {}
    # binary16 (src/half.cpp:9-50): 4096 values spanning normals, subnormals, overflow
    v = np.concatenate([rng.standard_normal(2048) * 300, rng.random(1024) * 2.0**-13, rng.standard_normal(1024) * 7e4])
    v = v.astype(np.float32)
    out["half_in"] = v
    out["half_bits"] = np.array([ref.ref_float_to_half_bits(float(x)) for x in v], np.uint16)
    # nms_greedy (src/postproc.cpp:47-63) keep lists
    for seed in range(6):
        r = np.random.default_rng(seed)
        n = 200
        xy = r.random((n, 2)) * 150
        wh = np.exp(r.uniform(np.log(4), np.log(60), (n, 2)))
        boxes = np.concatenate([xy, xy + wh], 1).astype(np.float32).astype(np.float64)
        scores = np.round(r.random(n), 2)
        keep = np.zeros(n, np.int64)
        nk = C.c_int64(0)
        assert ref.ref_nms_greedy(p(boxes), p(scores), None, n, 0.5, p(keep), C.byref(nk)) == 0
        out[f"nms{seed}_boxes"] = boxes.astype(np.float32)
        out[f"nms{seed}_scores"] = scores.astype(np.float32)
        out[f"nms{seed}_keep"] = keep[: nk.value]
    # update_scale trace (src/precision.cpp:45-56)
    ov = (rng.random(500) < 0.07).astype(np.int32)
    s, g = C.c_double(32768.0), C.c_int64(0)
    tr = []
    for o in ov:
        ref.ref_update_scale(C.byref(s), C.byref(g), 1, 13, 2.0, 0.5, 1.0, 2.0**20, int(o))
        tr.append((s.value, g.value))
    out["scale_overflow"] = ov
    out["scale_trace"] = np.array(tr, np.float64)
    # sgd_step_master (src/precision.cpp:84-100)
    n = 1000
    w = rng.standard_normal(n).astype(np.float32)
    vv = rng.standard_normal(n).astype(np.float32) * 0.1
    gg = rng.standard_normal(n).astype(np.float32)
    out["sgd_w0"], out["sgd_v0"], out["sgd_g"] = w.copy(), vv.copy(), gg
    assert ref.ref_sgd_step_master(p(w), p(vv), p(gg), n, 0.01, 0.9) == 0
    out["sgd_w1"], out["sgd_v1"] = w, vv
    np.savez_compressed(os.path.join(os.path.dirname(__file__), "reference_golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
