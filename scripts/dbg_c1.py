"""Debug helper: one C1-shaped graph_search batch (u8 d=128, 1024 queries) with a short timeout."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import datagen as D
from paper_1602_06819_b200 import KnngGraph
n0 = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
cfg = D.CONFIGS["C1"].with_sizes(n0=n0)
X = D.initial_points(cfg)
Q = D.stream_points(cfg, 0, 1024)
g = KnngGraph(X, cfg.k, device=0, capacity=n0 + 2000)
print("init ok", flush=True)
for it in range(3):
    ids, keys, st = g.search(Q, cfg.k, cfg.speedup, cfg.e_num, cfg.e_den, cfg.search_seed)
    print("search ok", it, st["search_evals"], st["ms_search"], flush=True)
first, st = g.insert_batch(Q, cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
print("insert ok", st["search_evals"], flush=True)
