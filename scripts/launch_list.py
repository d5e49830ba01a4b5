"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list into a
markdown table of per-kernel shares (usage: launch_list.py CSV TITLE CMD)."""
import csv, re, sys
from collections import OrderedDict
path, title, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = OrderedDict()
n = 0
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    v *= {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}.get(unit, 1)
    name = r[ki]
    m = re.search(r"(k_\w+)(<[^()]*>)?", name)
    key = (m.group(1) + (m.group(2) or "")) if m else name[:40]
    key = re.sub(r"unnamed>::|\(int\)|\(bool\)|cpddg::|<unnamed>::", "", key)
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += v
    n += 1
tot = sum(v[1] for v in agg.values())
print(f"# {title}\n\nCommand: `{cmd}`\n(after the same command exited 0 without ncu).  Serialised, cold-cache launches: compare SHARES.\n")
print(f"launches captured: {n} (unit ns)\n\n| kernel | launches | total ns | share | avg ns/launch |\n|---|---|---|---|---|")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {c} | {v:.0f} | {100 * v / tot:.1f}% | {v / c:.0f} |")
