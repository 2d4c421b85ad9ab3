"""aggregate the [sdb-prof] per-launch lines of SDB_PROFILE_VERBOSE=1 runs: python tools/prof_table.py LOG [filter]"""
import collections
import re
import sys

agg = collections.OrderedDict()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for l in open(sys.argv[1]):
    m = re.match(r"\[sdb-prof\] (\S+) (.*?)\s+([\d.]+) us\s+(\d+) TF/s\s+(\d+) GB/s", l)
    if not m or flt not in l:
        continue
    k = (m.group(1), m.group(2).strip())
    a = agg.setdefault(k, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += float(m.group(3))
rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
print("total us %.1f" % sum(v[1] for k, v in rows))
for k, v in rows[:50]:
    print("%-6s %-50s n=%2d %8.1f us  (%.1f each)" % (k[0], k[1], v[0], v[1], v[1] / v[0]))
