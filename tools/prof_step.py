"""One CUDA-event-instrumented eager C4 step after warm-up; with
SDB_PROFILE_VERBOSE=1 every launch group is printed to stderr as
[sdb-prof] <label> <us> <TF/s> <GB/s> (aggregate with tools/prof_table.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_05831_b200 import detector as D  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
p = D.preset(cfg)
det = D.Detector(p)
for i in range(3):
    det.feed(D.batch_slots(i + 1, 0, 1, p.batch))
    det.step()
det.losses()
prof = det.profile()
for k, v in prof.items():
    print("%-14s %8.3f ms  %8.1f TF/s  %8.1f GB/s  launches %d" % (k, v[0], v[1] / max(v[0], 1e-9) / 1e9,
                                                                  v[2] / max(v[0], 1e-9) / 1e6, v[3]))
det.close()
