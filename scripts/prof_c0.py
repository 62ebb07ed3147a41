"""C0 (B = 1) cycle breakdown: KNNG_LIB=.../libknng_prof.so KNNG_PROFILE=1 python scripts/prof_c0.py
(graph_insert_sequential of 32 points, the bench's step, after 3 warm-up steps; the library prints the K1
per-task counters).  Measurement only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen as D  # noqa: E402
from paper_1602_06819_b200 import KnngGraph  # noqa: E402

cfg = D.CONFIGS["C0"]
X = D.initial_points(cfg)
S = D.stream_points(cfg, 0, 200)
g = KnngGraph(X, cfg.k, capacity=cfg.n0 + 256)
pos = 0
for it in range(5):
    print("step", it, file=sys.stderr, flush=True)
    _, st = g.insert_sequential(S[pos:pos + 32], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
    pos += 32
    print({k: st[k] for k in ("search_evals", "search_starts", "search_expansions", "ball_nodes", "ms_search",
                              "ms_total")}, file=sys.stderr, flush=True)
