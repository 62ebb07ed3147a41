"""Small end-to-end case for compute-sanitizer (memcheck / racecheck / synccheck): every kernel of the
library runs at least once (u8 + f32 + Jaccard; init, search, insert, partition, staged multi-rank)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import datagen as D
from paper_1602_06819_b200 import KnngGraph
from paper_1602_06819_b200.dist import insert_batch_staged

for name, n0, B in (("C0", 700, 64), ("C2", 600, 64), ("C4", 400, 48)):
    cfg = D.CONFIGS[name].with_sizes(n0=n0)
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, 3 * B)
    Q = D.query_points(cfg, 32)
    g = KnngGraph(X, cfg.k, capacity=n0 + 4 * B)
    g.search(Q, cfg.k, 3.0, cfg.e_num, cfg.e_den, 1)
    g.insert_batch(S[:B], 3.0, cfg.e_num, cfg.e_den, cfg.depth, 1)
    for i in range(3):                          # B = 1 fast path (fused one-warp update)
        g.insert_batch(S[B + i:B + i + 1], 3.0, cfg.e_num, cfg.e_den, cfg.depth, 1)
    g.search(Q, cfg.k, 3.0, 1, 0, 1, full_scan=1)   # GNNS walk
    g.partition_kmedoids(4, 1.05, 2, 3)
    g.insert_batch(S[B + 3:2 * B], 3.0, cfg.e_num, cfg.e_den, cfg.depth, 1)
    g.search(Q, cfg.k, 3.0, cfg.e_num, cfg.e_den, 1, route=1)   # routing variant
    g.recompute_medoids(3, 0)
    reps = [KnngGraph(X, cfg.k, capacity=n0 + 4 * B) for _ in range(2)]
    for r in reps:
        r.partition_kmedoids(4, 1.05, 2, 3)
    insert_batch_staged(reps, [0, 1], 2, S[2 * B:3 * B], 3.0, cfg.e_num, cfg.e_den, cfg.depth, 1, 4)
    torch.cuda.synchronize()
    print(name, "ok", g.n)
print("sanitize case done")
