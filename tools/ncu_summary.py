"""Summarise an ncu report: key metrics, stall breakdown, instruction mix, top stalled SASS.
usage: python tools/ncu_summary.py report.ncu-rep [points] [json_out]"""
import csv
import io
import json
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
npts = float(sys.argv[2]) if len(sys.argv) > 2 else 0
out_json = sys.argv[3] if len(sys.argv) > 3 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
h = det[0]
keep = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "Achieved Active Warps Per SM", "L2 Hit Rate", "Registers Per Thread", "Grid Size", "Block Size",
        "Executed Ipc Active", "Avg. Active Threads Per Warp", "Theoretical Occupancy", "SM Frequency")
summary = {}
for row in det[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in keep and d.get("Metric Name") not in summary:
        summary[d["Metric Name"]] = (d.get("Metric Value"), d.get("Metric Unit"))
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
rh, ru, rv = raw[0], raw[1], raw[2]
rawd = dict(zip(rh, rv))
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "gpu__time_duration.sum"):
    if k in rawd:
        summary[k] = (rawd[k], ru[rh.index(k)])

def rawf(k):
    return float(str(rawd.get(k, "0")).replace(",", "") or 0)


# Cell-index lookup hit rates.  The point stream arrives by TMA with an L2 evict_first policy; the only
# evict_normal reads from the SMs are the index lookups (root / node / owner-pool loads), so the
# evict_normal read sectors at L2 are the index traffic.  In L1 the global loads are the index loads.
ih = rawf("lts__t_sectors_srcunit_tex_op_read_evict_normal_lookup_hit.sum")
im = rawf("lts__t_sectors_srcunit_tex_op_read_evict_normal_lookup_miss.sum")
lh = rawf("l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum")
lm = rawf("l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum")
index = {}
if ih + im > 0:
    index = {"index_l2_hit_rate": ih / (ih + im), "index_l1_hit_rate": lh / (lh + lm) if lh + lm else None,
             "index_l2_sectors_per_point": (ih + im) / npts if npts else None}
    red = rawf("lts__t_sectors_srcunit_tex_op_red.sum")
    if npts:
        index["red_sectors_per_point"] = red / npts
        index["l1_load_sectors_per_point"] = (lh + lm) / npts  # the SM-side random requests (index loads)
        summary["index lookups: L1 sectors per point"] = (f"{(lh + lm) / npts:.3f}", "")
        summary["global REDs: L2 sectors per point"] = (f"{red / npts:.3f}", "")
    summary["index lookups: L2 hit rate"] = (f"{100 * ih / (ih + im):.2f}", "%")
    if lh + lm:
        summary["index lookups: L1 hit rate"] = (f"{100 * lh / (lh + lm):.2f}", "%")
    if npts:
        summary["index lookups: L2 sectors per point"] = (f"{(ih + im) / npts:.3f}", "")
for k, (v, u) in summary.items():
    print(f"{k:40s} {v} {u}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
sh = src[1]
data = [dict(zip(sh, r)) for r in src[2:]]
cols = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: sum(float(d[c] or 0) for d in data) for c in cols}
T = sum(tot.values()) or 1
print("-- stall breakdown")
for c, v in sorted(tot.items(), key=lambda x: -x[1])[:8]:
    print(f"  {c:26s} {v / T * 100:5.1f}%")
cnt = Counter()
for d in data:
    ex = float(d["Instructions Executed"] or 0)
    toks = d["Source"].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    cnt[op.split(".")[0]] += ex
E = sum(cnt.values())
if npts:
    print(f"-- {E * 32 / npts:.1f} thread-instructions per point")
    for k, v in cnt.most_common(16):
        print(f"  {k:10s} {v * 32 / npts:6.2f}/pt")
key = "Warp Stall Sampling (All Samples)"
S = sum(float(d[key] or 0) for d in data) or 1
print("-- top stalled instructions")
for d in sorted(data, key=lambda d: -float(d[key] or 0))[:12]:
    print(f"  {float(d[key]) / S * 100:5.1f}%  {d['Source'][:90]}")
if out_json:
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def nbytes(k):  # ncu prints each metric in its own unit (e.g. Gbyte for reads, Mbyte for writes)
        if k not in rawd:
            return 0.0
        return float(str(rawd[k]).replace(",", "") or 0) * scale.get(ru[rh.index(k)], 1.0)

    dr = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
    with open(out_json, "w") as f:
        json.dump({"report": rep, "metrics": {k: v for k, (v, u) in summary.items()},
                   "dram_bytes_per_launch": dr, "points": npts,
                   "dram_bytes_per_point": dr / npts if npts else None, **index,
                   "stalls": {k: v / T for k, v in tot.items()}}, f, indent=1)
