"""Summarise the ncu outputs brought back in gpurun_out/ into profiles/ (tracked).

usage: python scripts/summarize_profiles.py <tag> [<config tag> [<launches.csv> [<k_search .ncu-rep>]]]
  reads the ncu --metrics gpu__time_duration.sum launch list and the ncu --set full capture of one
  k_search launch, writes profiles/<tag>_<cfg>_launches.md, profiles/<tag>_<cfg>_k_search_full.md
  and profiles/k_search_ncu_<cfg>.json (the DRAM bytes bench.py reports as roofline.traffic)
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "round1"
cfgtag = sys.argv[2] if len(sys.argv) > 2 else "C1"
lpath = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", "launches.csv")
rep = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "gpurun_out", "prof_search.ncu-rep")
out = os.environ.get("PROFILES_OUT") or os.path.join(ROOT, "profiles")
os.makedirs(out, exist_ok=True)

# ---- launch list ----
rows = list(csv.reader(open(lpath)))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h, start = r, i + 1
        break
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
agg = collections.defaultdict(list)
for r in rows[start:]:
    if len(r) > iv:
        agg[r[ik].split("(")[0]].append(float(r[iv].replace(",", "")) * scale[r[iu]])
tot = sum(sum(v) for v in agg.values())
lines = ["# %s %s: ncu launch list (`gpu__time_duration.sum`, --clock-control none)" % (tag, cfgtag), "",
         "Command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config %s "
         "--steps 2 --warmup 3 --no-cpu-baseline`" % cfgtag,
         "(whole program: graph_init + 5 insert batches + the e2e pass + torch recall).  Per-launch times are",
         "cold-cache and serialised; compare shares, not absolutes.", "",
         "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lines.append("| `%s` | %d | %.1f | %.1f | %.1f%% |" % (k, len(v), sum(v), sum(v) / len(v), 100 * sum(v) / tot))
# share of the insert step only: our kernels, minus the setup launches (graph_init's exact build
# and the partitioner: the launches of a kernel far longer than its median)
step = {}
for k, v in agg.items():
    if not (k.startswith("void knng::") or k.startswith("knng::")):
        continue
    med = sorted(v)[len(v) // 2]
    keep = [x for x in v if x <= 20 * med] if len(v) > 2 else v
    if "exact_build" in k or "medoid" in k or "greedy" in k or "bfs" in k.lower():
        continue
    if keep:
        step[k] = keep
st = sum(sum(v) for v in step.values())
lines += ["", "Share of one insert step (our kernels, graph_init excluded):", "",
          "| kernel | mean us | share of step |", "|---|---|---|"]
for k, v in sorted(step.items(), key=lambda kv: -sum(kv[1])):
    lines.append("| `%s` | %.1f | %.1f%% |" % (k, sum(v) / len(v), 100 * sum(v) / st))
open(os.path.join(out, "%s_%s_launches.md" % (tag, cfgtag)), "w").write("\n".join(lines) + "\n")

# ---- full capture of k_search ----
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hh, units, vals = r[0], r[1], r[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "l1tex__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__average_warp_latency_per_inst_issued.ratio", "lts__t_sector_hit_rate.pct"]
    got = {}
    md = ["# %s %s: `ncu --set full` of k_search (one launch of the bench step)" % (tag, cfgtag), "",
          "| metric | unit | value |", "|---|---|---|"]
    for i, x in enumerate(hh):
        if x in want or x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued"):
            md.append("| %s | %s | %s |" % (x, units[i], vals[i]))
            got[x] = (units[i], vals[i])

    def val(name, unit_scale):
        u, v = got[name]
        v = float(v.replace(",", ""))
        return v * unit_scale.get(u, 1.0)

    bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = val("dram__bytes_read.sum", bscale) + val("dram__bytes_write.sum", bscale)
    tscale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
    ms = val("gpu__time_duration.sum", tscale)
    json.dump({"kernel": "k_search", "config": cfgtag, "dram_bytes_per_launch": dram, "ms": ms,
               "source": "ncu --set full, " + tag},
              open(os.path.join(out, "k_search_ncu_%s.json" % cfgtag), "w"), indent=1)
    md += ["", "DRAM traffic per launch: %.1f MB." % (dram / 1e6), "",
           "Warp-stall samples and executed instructions per source line (top 30):", "", "```"]
    md += subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_lines.py"), rep, "30"],
                         capture_output=True, text=True).stdout.splitlines()
    md += ["```"]
    open(os.path.join(out, "%s_%s_k_search_full.md" % (tag, cfgtag)), "w").write("\n".join(md) + "\n")
print("wrote profiles/%s_%s_*" % (tag, cfgtag))
