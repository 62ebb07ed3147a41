"""Measurement helper: K1 (graph_search over one batch of stream points) under producer-shape
knobs (KNNG_NPROD / KNNG_STAGES / KNNG_LANE_EVAL / KNNG_RING / KNNG_SMEM_BITS), one graph per config.
Every setting must return the same ids/keys (the knobs change the schedule, not the result).
usage: python scripts/sweep_search.py C2 [--n0 N] [--reps R] [--settings "plan/RING=16/STAGES=4,NPROD=2"] (settings separated by /)"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--n0", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--kmedoids-iters", type=int, default=2)
    ap.add_argument("--settings", default="plan/RING=16/RING=32/SMEM_BITS=0/SMEM_BITS=1/STAGES=4/NPROD=2")
    args = ap.parse_args()
    import torch
    from paper_1602_06819_b200 import KnngGraph
    cfg = D.CONFIGS[args.config]
    if args.n0:
        cfg = cfg.with_sizes(n0=args.n0)
    X = D.initial_points(cfg)
    Q = D.stream_points(cfg, 0, cfg.batch)
    t0 = time.perf_counter()
    g = KnngGraph(X, cfg.k, device=0, capacity=cfg.n0 + cfg.batch + 8)
    if cfg.P:
        g.partition_kmedoids(cfg.P, cfg.imbalance, args.kmedoids_iters, cfg.part_seed)
    print("setup %.1f s" % (time.perf_counter() - t0), flush=True)
    if cfg.metric != D.JAC:
        Q = torch.from_numpy(Q).cuda()
    ref = None
    knobs = ("KNNG_NPROD", "KNNG_STAGES", "KNNG_LANE_EVAL", "KNNG_RING", "KNNG_SMEM_BITS", "KNNG_LEAN", "KNNG_WALK_PREFETCH", "KNNG_EX_ONE", "KNNG_WIN_PREFETCH")
    for s in args.settings.split("/"):
        for kn in knobs:
            os.environ.pop(kn, None)
        if s != "plan":
            for kv in s.split(","):
                kk, vv = kv.split("=")
                os.environ["KNNG_" + kk] = vv
        ms = []
        for _ in range(args.reps):
            oi = torch.empty((cfg.batch, cfg.k), dtype=torch.int32, device="cuda")
            ok = torch.empty((cfg.batch, cfg.k), dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            t = time.perf_counter()
            _, _, st = g.search(Q, cfg.k, cfg.speedup, cfg.e_num, cfg.e_den, cfg.search_seed, out=(oi, ok))
            torch.cuda.synchronize()
            ms.append(1000 * (time.perf_counter() - t))
        res = (oi.cpu().numpy(), ok.cpu().numpy())
        same = ref is None or (np.array_equal(ref[0], res[0]) and np.array_equal(ref[1], res[1]))
        ref = ref or res
        ev = st["search_evals"]
        V = {D.U8: cfg.dim, D.F32: 4 * cfg.dim, D.JAC: 118}[cfg.metric]
        gbs = (ev * (V + 4) + st["search_expansions"] * 4 * cfg.k) / (min(ms) / 1000) / 1e9
        print("%-4s %-22s %8.2f ms (min of %d)  alg %.0f GB/s  same=%s" % (
            args.config, s, min(ms), args.reps, gbs, same), flush=True)
    g.close()


if __name__ == "__main__":
    main()
