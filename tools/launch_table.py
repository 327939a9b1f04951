"""Launch list (ncu --metrics gpu__time_duration.sum --csv) -> per-kernel share table + JSON.
usage: python tools/launch_table.py launches.csv out.txt out.json"""
import csv
import json
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
tot = OrderedDict()
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0].split("<")[0]
    k = k.replace("void ", "").replace("rb::", "")
    n, t = tot.get(k, (0, 0.0))
    tot[k] = (n + 1, t + float(d["Metric Value"].replace(",", "")) / 1e3)
T = sum(t for _, t in tot.values()) or 1
lines = ["kernel                      launches  total_us   share   per_launch_us (cold-cache, serialised)"]
js = {}
for k, (n, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
    lines.append(f"{k:26s} {n:9d} {t:9.1f} {100 * t / T:6.1f}%   {t / n:9.1f}")
    js[k] = {"launches": n, "total_us": round(t, 1), "share": round(t / T, 4), "per_launch_us": round(t / n, 1)}
open(sys.argv[2], "w").write("\n".join(lines) + "\n")
json.dump(js, open(sys.argv[3], "w"), indent=1)
print("\n".join(lines))
