"""Summarise an ncu launch-list CSV (gpu__time_duration.sum, optionally dram bytes) as a markdown
table of per-kernel launches, time and share of the profiled steps.
usage: python tools/launch_summary.py <launches.csv> [title] [--ours]
--ours: only libsketchmp.so's kernels (drops torch's input-generation kernels, which run before
the timed region)."""
import collections
import csv
import sys

path = sys.argv[1]
args = [a for a in sys.argv[2:] if not a.startswith("--")]
title = args[0] if args else path
ours = "--ours" in sys.argv
rows = list(csv.reader(open(path)))
start = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
iN, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
iID = h.index("ID") if "ID" in h else None
per = collections.defaultdict(lambda: collections.defaultdict(float))
launch_names = {}
for r in rows[start + 1:]:
    if len(r) <= iV:
        continue
    try:
        v = float(r[iV].replace(",", ""))
    except ValueError:
        continue
    if ours and (r[iN].startswith("void at::") or r[iN].startswith("at::") or "at::native" in r[iN]):
        continue
    name = r[iN].split("(")[0]
    name = name.replace("void ", "").replace("skmp::", "").replace("<unnamed>::", "").replace("unnamed>::", "").split("<")[0]
    key = r[iID] if iID is not None else len(launch_names)
    launch_names[key] = name
    per[key][r[iM]] += v
agg = collections.defaultdict(lambda: collections.Counter())
for key, ms in per.items():
    a = agg[launch_names[key]]
    a["n"] += 1
    for m, v in ms.items():
        a[m] += v
tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
print(f"# {title}\n")
has_dram = any("dram__bytes_read.sum" in a for a in agg.values())
print("| kernel | launches | time (us) | share |" + (" DRAM GB |" if has_dram else ""))
print("|---|---|---|---|" + ("---|" if has_dram else ""))
for name, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    t = a["gpu__time_duration.sum"]
    line = f"| {name} | {a['n']} | {t / 1e3:.1f} | {t / tot:.4f} |"
    if has_dram:
        line += f" {(a['dram__bytes_read.sum'] + a['dram__bytes_write.sum']) / 1e9:.3f} |"
    print(line)
print(f"| total | {sum(a['n'] for a in agg.values())} | {tot / 1e3:.1f} | 1 |" + (" |" if has_dram else ""))
