#!/usr/bin/env python
"""The paper's parameter studies on the synthetic stand-ins, run through the C ABI
on the GPU.  Writes a markdown table + JSON under profiles/round2/.

  F1  expansion sweep (Fig. 1): recall@k of graph_search vs e at a fixed speedup
  F2  iGNNS vs GNNS (Fig. 2): recall@k vs speedup (= equal similarity budgets n/speedup);
      GNNS = full neighbour scan + no restart skipping (knng_params.full_scan = 1, e = inf)
  F3  update depth (Fig. 3): inserts with DEPTH 1..4 -> recall of the inserted rows,
      correct edges over all nodes, update similarities per insert
  F4  partition count (Fig. 4): partitioned search recall vs P at a fixed speedup
  F5  medoid recomputation interval (Fig. 5): graph quality after a stream with medoids
      recomputed every x% of it (graph_recompute_medoids) vs never

Recall ground truth: exact k-nn by brute force (torch on the GPU for vectors; the library's own search
at speedup 1 -- budget = pool, parity-tested equal to linear search -- for token sets).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen as D  # noqa: E402


def exact_knn(cfg, pts, queries, k, g=None, exclude=None):
    import torch
    if cfg.metric == D.JAC:
        ids, _, _ = g.search(queries, k + (1 if exclude is not None else 0), 1.0, 1, 0, 1)
        if exclude is None:
            return ids
        return np.stack([[x for x in r if x != e][:k] for r, e in zip(ids, exclude)])
    q = torch.from_numpy(np.asarray(queries)).cuda().float()
    bd = torch.full((len(q), k), float("inf"), device="cuda")
    bi = torch.zeros((len(q), k), dtype=torch.int64, device="cuda")
    ex = None if exclude is None else torch.from_numpy(np.asarray(exclude)).cuda()
    for i in range(0, len(pts), 1 << 19):
        blk = torch.from_numpy(pts[i:i + (1 << 19)]).cuda().float()
        d2 = torch.cdist(q, blk).pow(2)
        if ex is not None:
            cols = torch.arange(i, i + d2.shape[1], device="cuda")
            d2[ex[:, None] == cols[None, :]] = float("inf")
        vd, vi = torch.topk(d2, min(k, d2.shape[1]), largest=False)
        bd, sel = torch.topk(torch.cat([bd, vd], 1), k, largest=False)
        bi = torch.gather(torch.cat([bi, vi + i], 1), 1, sel)
    return bi.cpu().numpy()


def recall(got, exact):
    k = exact.shape[1]
    return float(np.mean([len(set(a.tolist()) & set(b.tolist())) / k for a, b in zip(got, exact)]))


def main():
    from paper_1602_06819_b200 import KnngGraph
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C4")
    ap.add_argument("--n0", type=int, default=100_000)
    ap.add_argument("--nq", type=int, default=1000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "round2", "sweeps"))
    args = ap.parse_args()
    rows = []
    for name in args.configs.split(","):
        cfg = D.CONFIGS[name].with_sizes(n0=min(args.n0, D.CONFIGS[name].n0))
        X = D.initial_points(cfg)
        Q = D.query_points(cfg, args.nq, seed_offset=7)
        t0 = time.time()
        g = KnngGraph(X, cfg.k, capacity=cfg.n0 + 20000)
        t_init = time.time() - t0
        ex = exact_knn(cfg, X, Q, cfg.k, g)
        tag = "%s n0=%d" % (name, cfg.n0)
        # F1: expansion sweep at the config's speedup
        for num, den in ((1, 1), (11, 10), (6, 5), (3, 2), (2, 1), (5, 1), (1, 0)):
            ids, _, st = g.search(Q, cfg.k, cfg.speedup, num, den, 5)
            rows.append(dict(study="F1 expansion", workload=tag, e="inf" if den == 0 else "%g" % (num / den),
                             speedup=cfg.speedup, algo="iGNNS", recall=recall(ids, ex),
                             sims_per_query=st["search_evals"] / len(Q),
                             skipped_per_query=st["search_skipped"] / len(Q)))
        # F2: iGNNS vs GNNS at equal budgets
        for sp in (2, 4, 8, 16, 32, 64, 128):
            for algo, fs, num, den in (("iGNNS", 0, cfg.e_num, cfg.e_den), ("GNNS", 1, 1, 0)):
                ids, _, st = g.search(Q, cfg.k, sp, num, den, 5, full_scan=fs)
                rows.append(dict(study="F2 iGNNS vs GNNS", workload=tag, e="%g" % (num / den) if den else "inf",
                                 speedup=sp, algo=algo, recall=recall(ids, ex),
                                 sims_per_query=st["search_evals"] / len(Q),
                                 expansions_per_query=st["search_expansions"] / len(Q)))
        g.close()
        # F3: update depth
        S = D.stream_points(cfg, 0, 8192)
        allp = None if cfg.metric == D.JAC else np.concatenate([X, S])
        for depth in (1, 2, 3, 4):
            g = KnngGraph(X, cfg.k, capacity=cfg.n0 + 8200)
            ball = 0
            for b0 in range(0, 8192, 1024):
                _, st = g.insert_batch(S[b0:b0 + 1024], cfg.speedup, cfg.e_num, cfg.e_den, depth, cfg.search_seed)
                ball += st["ball_nodes"]
            rs = np.random.default_rng(9)
            new = cfg.n0 + np.sort(rs.choice(8192, 300, replace=False))
            old = np.sort(rs.choice(cfg.n0, 300, replace=False))
            nodes = np.concatenate([new, old])
            if cfg.metric == D.JAC:
                qs = [X[i] if i < cfg.n0 else S[i - cfg.n0] for i in nodes]
                exr = exact_knn(cfg, None, qs, cfg.k, g, exclude=nodes)
            else:
                exr = exact_knn(cfg, allp, allp[nodes], cfg.k, exclude=nodes)
            got, _ = g.rows()
            rows.append(dict(study="F3 update depth", workload=tag, depth=depth,
                             recall_inserted=recall(got[new], exr[:300]), correct_edges=recall(got[old], exr[300:]),
                             update_sims_per_insert=ball / 8192))
            g.close()
        print("%s done (init %.1f s)" % (tag, t_init), file=sys.stderr, flush=True)
    # F4 partition count, routing variant (Q18), F5 medoid recomputation interval: the C3 recipe (u8 d=128)
    cfg = D.CONFIGS["C3"].with_sizes(n0=min(args.n0, 100_000))
    X = D.initial_points(cfg)
    Q = D.query_points(cfg, args.nq, seed_offset=7)
    tag = "C3 recipe n0=%d" % cfg.n0
    g0 = KnngGraph(X, cfg.k)
    ex = exact_knn(cfg, X, Q, cfg.k)
    ids, _, st = g0.search(Q, cfg.k, cfg.speedup, cfg.e_num, cfg.e_den, 5)
    rows.append(dict(study="F4 partition count", workload=tag, P=0, speedup=cfg.speedup, recall=recall(ids, ex),
                     routed_recall=None, sims_per_query=st["search_evals"] / len(Q)))
    g0.close()
    for P in (1, 2, 4, 8, 16):
        g = KnngGraph(X, cfg.k)
        g.partition_kmedoids(P, cfg.imbalance, 10, cfg.part_seed)
        ids, _, st = g.search(Q, cfg.k, cfg.speedup, cfg.e_num, cfg.e_den, 5)
        rid, _, rst = g.search(Q, cfg.k, cfg.speedup, cfg.e_num, cfg.e_den, 5, route=1)
        rows.append(dict(study="F4 partition count", workload=tag, P=P, speedup=cfg.speedup, recall=recall(ids, ex),
                         routed_recall=recall(rid, ex), sims_per_query=st["search_evals"] / len(Q),
                         routed_sims_per_query=rst["search_evals"] / len(Q)))
        g.close()
    # F5: a stream of as many inserts as the initial graph, medoids recomputed every 10% of the graph size
    n_ins = cfg.n0
    S = D.stream_points(cfg, 0, n_ins)
    allp = np.concatenate([X, S])
    for interval in (0.1, None):
        g = KnngGraph(X, cfg.k, capacity=cfg.n0 + n_ins + 8)
        g.partition_kmedoids(cfg.P, cfg.imbalance, 10, cfg.part_seed)
        pos, nxt, epoch, nrec = 0, (int(cfg.n0 * interval) if interval else None), 0, 0
        while pos < n_ins:
            B = min(cfg.batch, n_ins - pos)
            g.insert_batch(S[pos:pos + B], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
            pos += B
            if nxt is not None and pos >= nxt:
                g.recompute_medoids(cfg.part_seed, epoch)
                epoch += 1
                nrec += 1
                nxt = pos + int((cfg.n0 + pos) * interval)
        rs = np.random.default_rng(11)
        nodes = np.sort(rs.choice(cfg.n0 + n_ins, 1000, replace=False))
        exr = exact_knn(cfg, allp, allp[nodes], cfg.k, exclude=nodes)
        got, _ = g.rows()
        rows.append(dict(study="F5 medoid recomputation", workload=tag + " + %d inserts, P=%d" % (n_ins, cfg.P),
                         interval="every 10%" if interval else "never", recomputations=nrec,
                         correct_edges=recall(got[nodes], exr)))
        g.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(rows, open(args.out + ".json", "w"), indent=1)
    with open(args.out + ".md", "w") as f:
        f.write("# Parameter studies on the synthetic stand-ins (GPU, through the C ABI)\n\n")
        f.write("Generated by `scripts/sweeps.py`; recall@k against exact k-nn (brute force).\n\n")
        for study in sorted({r["study"] for r in rows}):
            rr = [r for r in rows if r["study"] == study]
            keys = [k for k in rr[0] if k != "study"]
            keys = list(dict.fromkeys(k for r in rr for k in r if k != "study"))
            f.write("## %s\n\n| %s |\n|%s\n" % (study, " | ".join(keys), "---|" * len(keys)))
            for r in rr:
                f.write("| %s |\n" % " | ".join(("%.4f" % r[k]) if isinstance(r.get(k), float) else str(r.get(k))
                                              for k in keys))
            f.write("\n")
    print(open(args.out + ".md").read())


if __name__ == "__main__":
    main()
