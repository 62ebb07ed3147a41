"""DESIGN.md results-table rows from bench.py JSON lines: python scripts/bench_table.py NAME=FILE ..."""
import json
import sys

print("| config | inserts/s | e2e inserts/s | K1 ms / step | K1 alg. bytes / HBM peak | similarities/s | "
      "recall@k (inserted) | correct edges | CPU oracle inserts/s |")
print("|---|---|---|---|---|---|---|---|---|")
for arg in sys.argv[1:]:
    name, f = arg.split("=", 1)
    d = None
    for ln in open(f):
        if ln.startswith("{"):
            d = json.loads(ln)
    if d is None:
        print("| %s | (no line) |" % name)
        continue
    cb = d.get("cpu_baseline")
    cpu = "%.0f (%d cores)" % (cb["value"], cb["cores"]) if cb else "—"
    r = d["roofline"]
    print("| %s | %.0f | %.0f | %.2f | %.1f%% | %.3g | %.3f | %.3f | %s |" % (
        name, d["value"], d["e2e"]["value"], r["ms_per_launch"], 100 * r["frac"], d.get("similarities_per_s", 0),
        d.get("recall_at_k") or 0, d["quality"]["correct_edge_fraction"], cpu))
