"""Group an ncu SASS source page into straight-line blocks by execution count:
usage: python tools/ncu_blocks.py src.csv points_per_iteration total_points [min_instr_per_iter]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:]]
it = float(sys.argv[3]) / float(sys.argv[2])
thr = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
blocks, cur = [], None


def op(src):
    t = src.split()
    if not t:
        return ""
    return (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]


tot = 0.0
for d in data:
    ex = float(d.get("Instructions Executed") or 0) / it
    tot += ex
    st = float(d.get("Warp Stall Sampling (All Samples)") or 0)
    thr_ex = float(d.get("Thread Instructions Executed") or 0) / it
    key = round(ex, 2)
    if cur and cur[0] == key:
        cur[2] += 1; cur[3] += st; cur[4].append(op(d["Source"])); cur[5] += thr_ex
    else:
        cur = [key, d["Address"], 1, st, [op(d["Source"])], thr_ex]
        blocks.append(cur)
S = sum(b[3] for b in blocks) or 1
print(f"warp instructions per iteration: {tot:.1f}")
for b in blocks:
    if b[0] * b[2] >= thr:
        c = Counter(b[4]).most_common(6)
        act = b[5] / max(b[0] * b[2], 1e-9)
        print(f"{b[1][-5:]} exec/it={b[0]:5.2f} n={b[2]:4d} instr/it={b[0] * b[2]:6.1f} act={act:4.1f} stall%={100 * b[3] / S:5.1f} {c}")
