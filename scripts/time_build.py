"""Measurement helper: graph_init (A0 exact build) wall time for a config with the tcgen05 path on
(default) and off (KNNG_TC=0), and whether the two graphs are identical.
usage: python scripts/time_build.py C1 [--n0 N] [--no-simt]"""
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
    ap.add_argument("--no-simt", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_1602_06819_b200 import KnngGraph
    cfg = D.CONFIGS[args.config]
    if args.n0:
        cfg = cfg.with_sizes(n0=args.n0)
    X = D.initial_points(cfg)
    res = {}
    for mode in (["1"] if args.no_simt else ["1", "0"]):
        os.environ["KNNG_TC"] = mode
        for rep in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            g = KnngGraph(X, cfg.k, device=0, capacity=cfg.n0 + 8)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            if rep == 1:
                res[mode] = g.rows()
            g.close()
        print("%s n0=%d KNNG_TC=%s graph_init %.3f s" % (cfg.name, cfg.n0, mode, dt), flush=True)
    if len(res) == 2:
        same = np.array_equal(res["1"][0], res["0"][0]) and np.array_equal(res["1"][1], res["0"][1])
        print("tcgen05 graph == SIMT graph:", same, flush=True)


if __name__ == "__main__":
    main()
