"""Summarise an ncu --csv launch list (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) of one step by kernel family:
    python tools/launch_summary.py launches.csv [conv_traffic.json] > summary.txt
The optional second argument writes the conv-family DRAM traffic that
bench.py reports as roofline.traffic."""
import json
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
    if len(sys.argv) > 2:
        conv = [m for k, m in per.items() if "conv_tma_kernel" in names[k] or "conv_tc_kernel" in names[k]]
        b = sum(m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0) for m in conv)
        with open(sys.argv[2], "w") as f:
            json.dump({"conv_launches_per_step": len(conv), "conv_dram_bytes_per_step": b,
                       "conv_dram_bytes_per_launch": b / max(len(conv), 1),
                       "conv_time_us_ncu": sum(m.get("gpu__time_duration.sum", 0.0) for m in conv) / 1e3,
                       "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                                 "--profile-from-start off over one C4 step (tools/one_step.py)"}, f, indent=1)
    print("# ncu launch list of one C4 training step (cold-cache, serialised; shares, not absolutes)")
    print("# kernels/step %d  sum %.1f us" % (len(per), tot))
    print("%9s %6s %4s %9s  kernel" % ("us", "share", "n", "DRAM MB"))
    for n, (t, c, b) in sorted(fam.items(), key=lambda kv: -kv[1][0]):
        print("%9.1f %6.3f %4d %9.1f  %s" % (t, t / tot, c, b, n))


if __name__ == "__main__":
    main()
