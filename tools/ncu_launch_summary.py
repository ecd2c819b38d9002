"""Share of GPU time per kernel from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file X.csv <cmd>`).

    python tools/ncu_launch_summary.py gpurun_out/r02_launches.csv [header line ...] > profiles/r02_launches_summary.txt
"""
import csv
import sys
from collections import defaultdict

import re

args = sys.argv[1:]
exclude = None
if args and args[0].startswith("--exclude="):
    exclude = re.compile(args.pop(0).split("=", 1)[1])
path, *header = args
rows = list(csv.reader(open(path)))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                  hdr.index("Metric Unit"))
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
         "s": 1e6}
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[start + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "").strip()
    if exclude is not None and exclude.search(name):
        continue
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
all_us = sum(tot.values())
for h in header:
    print(f"# {h}")
print(f"# {sum(cnt.values())} launches, {all_us:.1f} us of GPU time")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{cnt[k]:5d} launches {tot[k]:12.1f} us total {100 * tot[k] / all_us:6.2f}%  {k}")
