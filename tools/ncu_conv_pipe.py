"""Per-layer tensor-pipe utilisation of the C4 step's convolutions from ncu
counters (the north star's ">= 50 % tensor-pipe utilisation on backbone
convs"), as opposed to tools/conv_table.py's time-based TF/s.

  run:   one instrumented eager step (det.profile(): every conv launch sits in
         an NVTX range named by its layer shape) bracketed by
         cudaProfilerStart/Stop, for
           SDB_PROFILE_VERBOSE=1 ncu --nvtx --print-nvtx-rename kernel \
             --profile-from-start off --clock-control none --csv \
             --metrics gpu__time_duration.sum,\
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,\
dram__bytes_read.sum,dram__bytes_write.sum \
             --log-file launches.csv python tools/ncu_conv_pipe.py run [preset]
  table: python tools/ncu_conv_pipe.py table launches.csv
         per (part, pass, shape): launches, ncu time, tensor-pipe % of the
         elapsed cycles (time-weighted over the layer's launches), TF/s and
         DRAM bytes; backbone (stem, res2-res4, RPN) and RoI-head totals.
ncu times are cold-cache and serialised (every launch replayed alone): the
tensor-pipe fraction is the kernel's own; the step's shares come from
bench.py."""
import collections
import csv
import os
import re
import sys


def run(preset):
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1903_05831_b200 import detector as D
    p = D.preset(preset)
    det = D.Detector(p)
    for i in range(3):
        det.feed(D.batch_slots(i + 1, 0, 1, p.batch))
        det.step()
    det.losses()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    det.profile()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    det.close()


SHAPE = re.compile(r"(fprop|dgrad|wgrad)\S*\s+N(\d+) H(\d+) W(\d+) C(\d+) K(\d+) R(\d+) S(\d+) st(\d+)")


def table(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    iid, iname, imet, ival = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = collections.OrderedDict()
    names = {}
    for r in rows[1:]:
        per.setdefault(r[iid], {})[r[imet]] = float(r[ival].replace(",", ""))
        names[r[iid]] = r[iname]
    agg = collections.OrderedDict()
    for k, m in per.items():
        mt = SHAPE.search(names[k])
        # the renamed kernel reads "<NVTX range>/<function>": only the conv
        # launches themselves (a bucket's batched split-K reduce, issued inside
        # the last wgrad's range, is not tensor work)
        if not mt or "conv_t" not in names[k].split("/", 1)[-1]:
            continue
        kind = mt.group(1)
        N, H, W, C, K, R, S, st = (int(mt.group(i)) for i in range(2, 10))
        Ho = (H + 2 * (R // 2) - R) // st + 1
        Wo = (W + 2 * (S // 2) - S) // st + 1
        part = "head" if N >= 64 and H * W <= 196 else "backbone"
        a = agg.setdefault((part, kind, f"N{N} H{H} W{W} C{C} K{K} R{R} st{st}"), [0.0, 0.0, 0.0, 0.0])
        t = m.get("gpu__time_duration.sum", 0.0) / 1e3
        a[0] += t
        a[1] += t * m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0) / 100.0
        a[2] += (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / 1e6
        # a strided dgrad runs one launch per sub-pixel phase (st x st), everything else one per layer
        a[3] += 2.0 * N * Ho * Wo * K * C * R * S / (st * st if kind == "dgrad" else 1)
    tot = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    print("%-8s %-6s %-34s %8s %7s %7s %8s" % ("part", "pass", "shape", "ncu_us", "tensor", "TF/s", "DRAM_MB"))
    out = [(part, kind, shape, us, act, mb, fl) for (part, kind, shape), (us, act, mb, fl) in agg.items()]
    for part, kind, shape, us, act, mb, fl in sorted(out, key=lambda r: -r[3]):
        print("%-8s %-6s %-34s %8.1f %6.1f%% %7.0f %8.1f" % (part, kind, shape, us, 100 * act / us, fl / us / 1e6, mb))
        tot[part][0] += us
        tot[part][1] += act
        tot[part][2] += fl
    for part, (us, act, fl) in tot.items():
        print("TOTAL %-8s ncu %.1f us  tensor-pipe %.1f %% of elapsed cycles (time-weighted)  %.0f TF/s" %
              (part, us, 100 * act / us, fl / us / 1e6))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2] if len(sys.argv) > 2 else "c4")
    else:
        table(sys.argv[2])
