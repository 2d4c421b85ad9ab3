"""Summarise an ncu --csv launch list (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) of one step by kernel family:
    python tools/launch_summary.py launches.csv > summary.txt"""
import collections
import csv
import re
import sys


def main():
    lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    iid, iname, imet, ival = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[iid]][r[imet]] = float(r[ival].replace(",", ""))
        names[r[iid]] = r[iname]
    fam = collections.OrderedDict()
    for k, m in per.items():
        n = re.sub(r"\(.*", "", names[k]).replace("void ", "").replace("sdb::", "")
        n = re.sub(r"\(anonymous namespace\)::", "", n)
        f = fam.setdefault(n, [0.0, 0, 0.0])
        f[0] += m.get("gpu__time_duration.sum", 0.0) / 1e3
        f[1] += 1
        f[2] += (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / 1e6
    tot = sum(v[0] for v in fam.values())
    print("# ncu launch list of one C4 training step (cold-cache, serialised; shares, not absolutes)")
    print("# kernels/step %d  sum %.1f us" % (len(per), tot))
    print("%9s %6s %4s %9s  kernel" % ("us", "share", "n", "DRAM MB"))
    for n, (t, c, b) in sorted(fam.items(), key=lambda kv: -kv[1][0]):
        print("%9.1f %6.3f %4d %9.1f  %s" % (t, t / tot, c, b, n))


if __name__ == "__main__":
    main()
