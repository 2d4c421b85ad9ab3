"""Per-layer conv table from an SDB_PROFILE_VERBOSE=1 step (tools/prof_step.py
stderr): TF/s per (pass, shape), the FLOP-weighted backbone figure (stem,
res2-res4, RPN: the north star's ">= 50 % tensor-pipe on backbone convs")
against the measured peak, and each layer's roofline attainment
t_min / t with t_min = max(FLOP / peak_tc, algorithmic bytes / peak_hbm)
(fp16 operands and output once; the many thin 1x1 layers are HBM-bound).
python tools/conv_table.py LOG [peak_tflops] [peak_hbm_GBps]"""
import collections
import re
import sys

peak = float(sys.argv[2]) if len(sys.argv) > 2 else 1665.8
hbm = float(sys.argv[3]) if len(sys.argv) > 3 else 6458.4
rows = collections.OrderedDict()
for line in open(sys.argv[1]):
    m = re.match(r"\[sdb-prof\] (fprop\S*|dgrad\S*|wgrad)\s+N(\d+) H(\d+) W(\d+) C(\d+) K(\d+) R(\d+) S(\d+) st(\d+)\s+"
                 r"([\d.]+) us\s+(\d+) TF/s", line)
    if not m:
        continue
    kind = m.group(1).split("(")[0].replace("+res", "")
    N, H, W, C, K, R, S, st = (int(m.group(i)) for i in range(2, 10))
    us = float(m.group(10))
    Ho, Wo = (H + 2 * (R // 2) - R) // st + 1 if R > 1 else (H - 1) // st + 1, (W + 2 * (S // 2) - S) // st + 1 if S > 1 else (W - 1) // st + 1
    flop = 2.0 * N * Ho * Wo * K * C * R * S
    x_b, y_b, w_b = 2.0 * N * H * W * C, 2.0 * N * Ho * Wo * K, 2.0 * K * R * S * C
    byts = x_b + y_b + w_b + (x_b if "+res" in m.group(1) else 0.0)  # dgrad+res also reads the addend
    part = "head" if N >= 64 and H * W <= 196 else "backbone"
    key = (part, kind, f"N{N} H{H} W{W} C{C} K{K} R{R} st{st}")
    a = rows.setdefault(key, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += us
    a[2] += flop
    a[3] += max(flop / (peak * 1e12), byts / (hbm * 1e9)) * 1e6
tot = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
print("%-8s %-6s %-38s %3s %9s %8s %6s %7s" % ("part", "pass", "shape", "n", "us", "TF/s", "tc", "roofl"))
for (part, kind, shape), (n, us, fl, tmin) in sorted(rows.items(), key=lambda kv: -kv[1][1]):
    tf = fl / (us * 1e-6) / 1e12
    print("%-8s %-6s %-38s %3d %9.1f %8.0f %6.2f %7.2f" % (part, kind, shape, n, us, tf, tf / peak, tmin / us))
    tot[part][0] += us
    tot[part][1] += fl
    tot[part][2] += tmin
for part, (us, fl, tmin) in tot.items():
    tf = fl / (us * 1e-6) / 1e12
    print("TOTAL %-8s %9.1f us %8.3f TFLOP  %6.0f TF/s  tensor frac %.3f of %.0f  roofline attainment %.3f"
          % (part, us, fl / 1e12, tf, tf / peak, peak, tmin / us))
