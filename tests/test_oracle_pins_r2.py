"""Pins of the oracle's remaining open branches (round 2), against tests/pyref.py.

* iGNNS without the Q9 shortcut: the oracle restarts when a walk moves onto an already expanded
  node (reading Q9, "result-equivalent").  tests/pyref.py walks literally (keep moving to
  the first improving neighbour, re-scanning expanded rows on cached keys).  Results and the
  evals / starts / skipped counters must agree on random u8, f32 and Jaccard graphs, partitioned and
  not, for speedups 1.5..10 and e in {6/5, 1, 5, inf}.
* Alg. 4 with the sampled-candidate medoid update (reading Q22) -- exact_limit lowered so every
  cluster takes the sampled branch -- and with the exact branch, all three metrics, including the
  fp32 assign comparator, against an exact-fraction re-derivation.
"""
import numpy as np
import pytest

from oracle import oracle as O
import datagen as D
from tests import pyref as R


def _points(metric, rng, n, dim=4):
    if metric == O.U8:
        return rng.integers(0, 40, size=(n, dim)).astype(np.uint8)
    if metric == O.F32:   # integer-valued fp32 (|x| <= 6): every canonical-order sum is exact
        return rng.integers(-6, 7, size=(n, dim)).astype(np.float32)
    out = []
    for _ in range(n):
        L = int(rng.integers(2, 8))
        out.append(np.sort(rng.choice(25, size=L, replace=False)).astype(np.uint32))
    return out


def _graph(metric, n, k, seed):
    rng = np.random.default_rng(seed)
    X = _points(metric, rng, n)
    g = O.OracleGraph(metric, X, k=k)
    g.init_exact(2)
    return g, rng


@pytest.mark.parametrize("metric", [O.U8, O.F32, O.JAC])
def test_ignns_equals_literal_walk_without_q9_shortcut(metric):
    g, rng = _graph(metric, 260, 6, 1100 + metric)
    rows = g.ids[:g.n]
    moved_onto_expanded = 0
    for qi in range(60):
        q = _points(metric, rng, 1)[0]
        sp = float(rng.choice([1.5, 2.0, 3.0, 5.0, 10.0]))
        e_num, e_den = [(6, 5), (1, 1), (5, 1), (1, 0)][qi % 4]
        ids, keys, st = g.ignns(q, 6, sp, e_num, e_den, seed=11, pid=qi)
        rid, rkey, rst = R.ignns_literal(metric, g.point, rows, q, 6, sp, e_num, e_den, 11, qi)
        assert ids.tolist() == rid and keys.tolist() == rkey, (qi, ids, rid)
        assert (st["evals"], st["starts"], st["skipped"]) == (rst["evals"], rst["starts"], rst["skipped"])
        # the literal walk expands at least as many rows (it re-scans expanded ones)
        moved_onto_expanded += st["expansions"] < _literal_expansions(metric, g, rows, q, sp, e_num, e_den, qi)
    assert moved_onto_expanded > 0   # the shortcut branch was really exercised


def _literal_expansions(metric, g, rows, q, sp, e_num, e_den, qi):
    """Count row scans of the literal walk (instrumented copy of the pyref walk's expansions)."""
    count = [0]
    orig = rows

    class Rows:
        def __len__(self):
            return len(orig)

        def __getitem__(self, i):
            count[0] += 1
            return orig[i]
    R.ignns_literal(metric, g.point, Rows(), q, 6, sp, e_num, e_den, 11, qi)
    return count[0]


@pytest.mark.parametrize("metric", [O.U8, O.JAC])
def test_partitioned_ignns_equals_literal_walk(metric):
    g, rng = _graph(metric, 240, 5, 1200 + metric)
    part, med, _ = g.partition_kmedoids(4, 1.05, 3, 2)
    g.set_partition(part, med)
    rows = g.ids[:g.n]
    for qi in range(24):
        q = _points(metric, rng, 1)[0]
        p = qi % 4
        pool = np.nonzero(part == p)[0].astype(np.int32)
        ids, keys, st = g.ignns(q, 5, 2.5, 6, 5, seed=5, pid=qi, part=p, pool=pool)
        rid, rkey, rst = R.ignns_literal(metric, g.point, rows, q, 5, 2.5, 6, 5, 5, qi, pool=pool.tolist(), part=p)
        assert ids.tolist()[:len(rid)] == rid and keys.tolist()[:len(rkey)] == rkey
        assert (st["evals"], st["starts"], st["skipped"]) == (rst["evals"], rst["starts"], rst["skipped"])


def test_injected_starts_literal_walk():
    """W3-style injected starts on a random graph (the start_override hook of graph_search)."""
    g, rng = _graph(O.U8, 120, 4, 1300)
    rows = g.ids[:g.n]
    for qi in range(20):
        q = _points(O.U8, rng, 1)[0]
        starts = rng.integers(0, g.n, size=12).tolist()
        ids, keys, st = g.ignns(q, 4, 3.0, 6, 5, seed=0, pid=0, starts=starts)
        rid, rkey, rst = R.ignns_literal(O.U8, g.point, rows, q, 4, 3.0, 6, 5, 0, 0, starts=starts)
        assert ids.tolist()[:len(rid)] == rid and keys.tolist()[:len(rkey)] == rkey
        assert st["evals"] == rst["evals"] and st["skipped"] == rst["skipped"]


@pytest.mark.parametrize("metric", [O.U8, O.F32, O.JAC])
@pytest.mark.parametrize("exact_limit", [4096, 25])
def test_kmedoids_equals_exact_fraction_rederivation(metric, exact_limit):
    """exact_limit = 25 < every cluster: the Q22 sampled-candidate update on every cluster."""
    g, _ = _graph(metric, 200, 4, 1400 + metric)
    rows = g.ids[:g.n]
    for P, imb, seed in ((2, 1.0, 3), (4, 1.1, 9), (5, 1.05, 21)):
        part, med, cost = g.partition_kmedoids(P, imb, 6, seed, exact_limit=exact_limit, ncand=8)
        rpart, rmed, rcost = R.kmedoids(metric, g.point, rows, P, imb, 6, seed, exact_limit=exact_limit, ncand=8)
        assert part.tolist() == rpart
        assert med.tolist() == rmed
        assert cost.tolist() == rcost


def test_kmedoids_f32_assign_uses_the_capacity_weight():
    """fp32 assign: score = s(m,u) (1 - |C|/cap), s = 1/(1+D), compared exactly.
    1-D points, medoids x=0 (A) and x=10 (B), cap = ceil(8 * 1.5 / 2) = 6.  Hand trace, ascending id:
    x=0,1,2,-1,-2 -> A (A's sizes 0..4); x=10 -> B; x=4 (id 6): D_A = 16, D_B = 36, so the raw
    similarity prefers A, but score_A = 1/17 * 1/6 = 0.0098 < score_B = 1/37 * 5/6 = 0.0225 -> B;
    x=11 -> B.  A comparator with a dropped or transposed weight puts id 6 in A."""
    X = np.array([[0], [1], [2], [-1], [-2], [10], [4], [11]], np.float32)
    g = O.OracleGraph(O.F32, X, k=2)
    g.init_exact(1)
    part, med, cost = g.partition_kmedoids(2, 1.5, 1, 0, init_medoids=[0, 5])
    assert part.tolist() == [0, 0, 0, 0, 0, 1, 1, 1]
    rpart, rmed, rcost = R.kmedoids(O.F32, g.point, g.ids[:g.n], 2, 1.5, 1, 0, init=[0, 5])
    assert rpart == part.tolist() and rmed == med.tolist() and rcost == cost.tolist()


# ---------------------------------------------------------------------------
# GNNS baseline (section 2.2): full neighbour scan, move to the best neighbour
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("metric", [O.U8, O.F32, O.JAC])
def test_gnns_equals_literal_full_scan_walk(metric):
    g, rng = _graph(metric, 240, 6, 1500 + metric)
    rows = g.ids[:g.n]
    for qi in range(40):
        q = _points(metric, rng, 1)[0]
        sp = float(rng.choice([1.5, 3.0, 8.0]))
        e_num, e_den = [(1, 0), (6, 5)][qi % 2]     # GNNS proper (no skip) and the ablation with the skip rule
        ids, keys, st = g.ignns(q, 6, sp, e_num, e_den, seed=13, pid=qi, full_scan=1)
        rid, rkey, rst = R.ignns_literal(metric, g.point, rows, q, 6, sp, e_num, e_den, 13, qi, full_scan=True)
        assert ids.tolist() == rid and keys.tolist() == rkey, qi
        assert (st["evals"], st["starts"], st["skipped"]) == (rst["evals"], rst["starts"], rst["skipped"])


def test_gnns_hand_trace_differs_from_eager():
    """1-D u8 points 0,10,20,30,40 (k=2, rows as W1: 0:(1,2) 1:(0,2) 2:(1,3) 3:(2,4) 4:(3,2)),
    query 25 (D = 625, 225, 25, 25, 225), injected start [0], e = inf.
    iGNNS (eager): expand 0 -> 1 (225) improves, move; expand 1 -> 0 cached, 2 (25) move;
    expand 2 -> 1 cached, 3 (25) not strictly better: local maximum.  3 expansions, evals 0,1,2,3.
    GNNS: expand 0 -> evaluates 1 AND 2, moves to the best (2); expand 2 -> 3 (25) not better.
    2 expansions, same 4 evals.  Budget 2: both stop before evaluating 2 -> (225,1),(625,0)."""
    X = D.line_points([0, 10, 20, 30, 40])
    g = O.OracleGraph(O.U8, X, k=2)
    g.init_exact(1)
    q = np.array([25], np.uint8)
    for fs in (0, 1):
        i2, k2, s2 = g.ignns(q, 2, 2.5, 1, 0, seed=0, pid=0, starts=[0], full_scan=fs)   # budget floor(5/2.5) = 2
        assert [(int(a), int(b)) for a, b in zip(k2, i2)] == [(225, 1), (625, 0)] and s2["evals"] == 2
        i5, k5, s5 = g.ignns(q, 2, 1.0, 1, 0, seed=0, pid=0, starts=[0], full_scan=fs)   # budget 5
        assert [(int(a), int(b)) for a, b in zip(k5, i5)] == [(25, 2), (25, 3)] and s5["evals"] == 4
        assert s5["expansions"] == (2 if fs else 3)


def test_gnns_spec_examples():
    """SPEC gnns_search examples: unlimited budget -> recall 1.0 vs brute force; a query equal to a
    stored point is rank 1."""
    g, rng = _graph(O.U8, 90, 5, 1600)
    for qi in range(10):
        q = _points(O.U8, rng, 1)[0]
        ids, keys, st = g.ignns(q, 5, 1.0, 1, 0, seed=2, pid=qi, full_scan=1)
        want = sorted((R.metric_value(O.U8, q, g.point(u)), u) for u in range(g.n))[:5]
        assert [(int(a), int(b)) for a, b in zip(keys, ids)] == [(int(d), u) for d, u in want]
    for u in (0, 17, 89):
        ids, keys, st = g.ignns(g.point(u).copy(), 5, 2.0, 1, 0, seed=3, pid=u, full_scan=1, starts=[u])
        assert ids[0] == u and keys[0] == 0


# ---------------------------------------------------------------------------
# Alg. 5's medoid recomputation and the nearest-medoid routing variant (reading Q18)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("metric", [O.U8, O.JAC])
@pytest.mark.parametrize("exact_limit", [4096, 20])
def test_recompute_medoids_equals_rederivation(metric, exact_limit):
    g, rng = _graph(metric, 220, 4, 1700 + metric)
    g.cap = 400
    part, med, _ = g.partition_kmedoids(4, 1.05, 3, 2)
    g.set_partition(part, med)
    pts = _points(metric, rng, 60)
    g.insert_batch(pts if metric == O.JAC else np.stack(pts), 3.0, 6, 5, 2, 8)
    rows = g.ids[:g.n]
    for epoch in (0, 3):
        want, wcost = R.recompute_medoids(rows, g.part_of[:g.n], g.medoids, 17, epoch, exact_limit, 8)
        got, cost = g.recompute_medoids(17, epoch, exact_limit, 8)
        assert got.tolist() == want and cost == wcost


@pytest.mark.parametrize("metric", [O.U8, O.JAC])
def test_routed_search_equals_literal_walk_on_nearest_partition(metric):
    g, rng = _graph(metric, 240, 5, 1800 + metric)
    part, med, _ = g.partition_kmedoids(4, 1.05, 3, 2)
    g.set_partition(part, med)
    rows = g.ids[:g.n]
    qs = [_points(metric, rng, 1)[0] for _ in range(20)]
    qa = qs if metric == O.JAC else np.stack(qs)
    ids, keys, st = g.search(qa, 5, 2.5, 6, 5, 3, route=1)
    for i, q in enumerate(qs):
        p = R.nearest_medoid(metric, g.point, q, g.medoids)
        pool = np.nonzero(part == p)[0].tolist()
        rid, rkey, rst = R.ignns_literal(metric, g.point, rows, q, 5, 2.5, 6, 5, 3, i, pool=pool, part=p)
        assert ids[i].tolist()[:len(rid)] == rid and keys[i].tolist()[:len(rkey)] == rkey
        assert st[i, 0] == rst["evals"]


def test_routing_with_one_partition_is_unpartitioned():
    g, rng = _graph(O.U8, 150, 5, 1900)
    h, _ = _graph(O.U8, 150, 5, 1900)
    h.set_partition(np.zeros(150, np.uint8), np.array([0], np.int32))
    Q = np.stack(_points(O.U8, rng, 12))
    a = g.search(Q, 5, 4.0, 6, 5, 7)
    b = h.search(Q, 5, 4.0, 6, 5, 7, route=1)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all() and (a[2] == b[2]).all()
