#!/usr/bin/env python
"""K1 launch-plan A/B on one graph: build a config's graph once (plus Alg. 4 when partitioned), then
time graph_search of one batch of stream points under several knob settings (env vars read by the
launch plan on every call).  Results must be identical across settings (checked).  Measurement only."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n0", type=int, default=2_000_000)
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("settings", nargs="*", help="KEY=V[,KEY=V...] per setting; '-' = defaults")
    args = ap.parse_args()
    from paper_1602_06819_b200 import KnngGraph
    cfg = D.CONFIGS[args.config].with_sizes(n0=args.n0)
    X = D.initial_points(cfg)
    Q = D.stream_points(cfg, 0, args.nq or cfg.batch)
    t0 = time.time()
    g = KnngGraph(X, cfg.k)
    if cfg.P:
        g.partition_kmedoids(cfg.P, cfg.imbalance, 10, cfg.part_seed)
    print("setup %.1f s" % (time.time() - t0), flush=True)
    ref = None
    for sset in (args.settings or ["-"]):
        env = {} if sset == "-" else dict(kv.split("=") for kv in sset.split(","))
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        ms = []
        for _ in range(args.reps):
            ids, keys, st = g.search(Q, cfg.k, cfg.speedup, cfg.e_num, cfg.e_den, cfg.search_seed)
            ms.append(st["ms_search"])
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        same = None
        if ref is None:
            ref = (ids, keys)
        else:
            same = bool((ref[0] == ids).all() and (ref[1] == keys).all())
        V = cfg.dim if cfg.metric == D.U8 else 4 * cfg.dim
        gbs = (st["search_evals"] * (V + 4) + st["search_expansions"] * 4 * cfg.k) / (min(ms) / 1e3) / 1e9
        print(json.dumps({"setting": sset, "ms": [round(m, 3) for m in ms], "alg_GBps": round(gbs, 1),
                          "evals": st["search_evals"], "identical": same}), flush=True)


if __name__ == "__main__":
    main()
