"""Summarise an ncu --set full report: key raw metrics, then warp-stall samples per source line
(ncu -i REPORT --page source --csv --print-source cuda,sass)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
if len(raw) > 2:
    h, v = raw[0], raw[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "sm__inst_executed.avg.per_cycle_active", "launch__grid_size", "launch__registers_per_thread",
            "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    for i, n in enumerate(h):
        if n in want or ("pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued")):
            print("%-70s %s %s" % (n, v[i], raw[1][i]))
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                                      capture_output=True, text=True).stdout.splitlines()))
cur, hdr = None, None
agg = collections.defaultdict(lambda: [0, 0])
src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    d = dict(zip(hdr, r))
    try:
        ln = int(d["Line No"])
        agg[(cur, ln)][0] += int(float(d.get("Warp Stall Sampling (All Samples)") or 0))
        agg[(cur, ln)][1] += int(float(d.get("Instructions Executed") or 0))
    except ValueError:
        continue
    src[(cur, ln)] = r[1][:100]
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print("stall samples %d, instructions %d" % (tot, toti))
for k, v in sorted(agg.items(), key=lambda x: -x[1][int(__import__("os").environ.get("NCU_SORT_INST", "0"))])[:top]:
    print("%5.1f%% %5.1f%%  %s:%d  %s" % (100 * v[0] / tot, 100 * v[1] / toti, k[0], k[1], src.get(k, "")))
