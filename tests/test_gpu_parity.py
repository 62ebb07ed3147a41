"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on the same seeded inputs.

Bar: integer metrics bit-exact; fp32 every key within 1e-5 relative and
edge agreement >= 0.995 (north_star), which the canonical fp32 order makes bit-exact in practice.
"""
import math

import numpy as np
import pytest

import datagen as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu

F32_RTOL = 1e-5


def _graph(X, k, cap=None):
    from paper_1602_06819_b200 import KnngGraph
    return KnngGraph(X, k, device=0, capacity=cap or 2 * len(X))


def _assert_rows_equal(metric, gi, gk, oi, ok, what):
    if metric == O.F32:
        gv = np.asarray(gk).view(np.float32).astype(np.float64)
        ov = np.asarray(ok).view(np.float32).astype(np.float64)
        assert np.all(np.abs(gv - ov) <= F32_RTOL * np.maximum(np.abs(ov), 1e-30)), what + ": keys"
        agree = np.mean([len(set(a.tolist()) & set(b.tolist())) / len(b) for a, b in zip(gi, oi)])
        assert agree >= 0.995, "%s: edge agreement %.5f" % (what, agree)
        # canonical order: expect bit-exact
        assert (gi == oi).all() and (gk == ok).all(), what + ": not bit-exact (within tolerance)"
    else:
        bad = np.nonzero((gi != oi).any(1) | (gk != ok).any(1))[0]
        assert len(bad) == 0, "%s: %d rows differ, first %s: gpu %s %s oracle %s %s" % (
            what, len(bad), bad[:5], gi[bad[0]], gk[bad[0]], oi[bad[0]], ok[bad[0]])


def _cfg_small(name, **kw):
    return D.CONFIGS[name].with_sizes(**kw)


# ---------------------------------------------------------------------------
# A0 graph_init
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,n0,k", [("C0", 2000, 10), ("C1", 3000, 10), ("C2", 2500, 20)])
def test_graph_init_exact(name, n0, k):
    cfg = _cfg_small(name, n0=n0)
    X = D.initial_points(cfg)
    g = _graph(X, k)
    o = O.OracleGraph(cfg.metric, X, k)
    o.init_exact()
    gi, gk = g.rows()
    _assert_rows_equal(cfg.metric, gi, gk, o.ids[:n0], o.keys[:n0], "graph_init " + name)


@pytest.mark.parametrize("metric,dim", [(O.U8, 1), (O.U8, 3), (O.U8, 17), (O.F32, 1), (O.F32, 5), (O.F32, 33),
                                        (O.F32, 130), (O.U8, 300)])
def test_graph_init_ragged_dims_and_ties(metric, dim):
    rng = np.random.default_rng(dim + 10 * metric)
    n = 333   # ragged: not a multiple of the 64-row tile
    if metric == O.U8:
        X = rng.integers(0, 4, size=(n, dim)).astype(np.uint8)      # many exact ties
    else:
        X = rng.standard_normal((n, dim)).astype(np.float32)
    g = _graph(X, 7)
    o = O.OracleGraph(metric, X, 7)
    o.init_exact()
    gi, gk = g.rows()
    _assert_rows_equal(metric, gi, gk, o.ids[:n], o.keys[:n], "init d=%d" % dim)


@pytest.mark.parametrize("n,dim,k", [(129, 32, 1), (700, 128, 10), (555, 40, 16), (1300, 200, 32), (300, 256, 7),
                                     (2049, 8, 10)])
def test_graph_init_tcgen05_vs_oracle(n, dim, k):
    """u8 rows go through the tcgen05 kind::i8 kernel (d <= 256): ragged row/column tiles, odd chunk
    counts (padded K), top-k sizes 1..32 (KM = 10 / 16 / 32 instances), heavy ties."""
    rng = np.random.default_rng(n + dim)
    X = rng.integers(0, 6 if dim > 64 else 3, size=(n, dim)).astype(np.uint8)
    g = _graph(X, k)
    o = O.OracleGraph(O.U8, X, k)
    o.init_exact()
    gi, gk = g.rows()
    _assert_rows_equal(O.U8, gi, gk, o.ids[:n], o.keys[:n], "tc init n=%d d=%d k=%d" % (n, dim, k))


@pytest.mark.parametrize("n,dim,k,scale", [(129, 4, 1, 1.0), (700, 96, 20, 1.0), (555, 33, 16, 100.0),
                                           (1300, 96, 32, 0.01), (1300, 128, 32, 1.0), (300, 96, 7, 1.0)])
def test_graph_init_tcgen05_f32_vs_oracle(n, dim, k, scale):
    """fp32 rows go through the 3xTF32 tcgen05 screen + exact canonical rerank (d <= 128): the graph
    must be bit-identical to the oracle's, including near-ties (duplicated points, tiny offsets)."""
    rng = np.random.default_rng(n + dim)
    X = (rng.standard_normal((n, dim)) * scale).astype(np.float32)
    X[n // 2:n // 2 + 20] = X[:20]                                  # exact duplicates (key 0, ties by id)
    X[n // 3:n // 3 + 20] = X[:20] + np.float32(1e-6 * scale)       # near-duplicates
    g = _graph(X, k)
    o = O.OracleGraph(O.F32, X, k)
    o.init_exact()
    gi, gk = g.rows()
    _assert_rows_equal(O.F32, gi, gk, o.ids[:n], o.keys[:n], "tc f32 init n=%d d=%d k=%d" % (n, dim, k))


def test_graph_init_errors():
    from paper_1602_06819_b200 import KnngGraph, KnngError
    with pytest.raises(KnngError) as e:
        KnngGraph(np.zeros((5, 4), np.uint8), 5)
    assert e.value.code == -2
    with pytest.raises(KnngError) as e:
        KnngGraph(np.zeros((50, 4), np.uint8), 0)
    assert e.value.code == -1
    with pytest.raises(KnngError) as e:
        KnngGraph(np.zeros((50, 4), np.uint8), 33)
    assert e.value.code == -1


# ---------------------------------------------------------------------------
# A2/A3 graph_search
# ---------------------------------------------------------------------------
def test_search_w3_hand_traces():
    X = D.line_points([0, 10, 20, 30, 40, 100, 110, 120])
    g = _graph(X, 2)
    q = D.line_points([33])
    ids, keys, st = g.search(q, 2, 1.0, 6, 5, 0, starts=[1, 6, 7, 5])
    assert [(int(a), int(b)) for a, b in zip(keys[0], ids[0])] == [(9, 3), (49, 4)]
    assert st["search_evals"] == 8 and st["search_skipped"] == 3
    ids, keys, st = g.search(q, 2, 2.0, 6, 5, 0, starts=[1, 6, 7, 5])
    assert [(int(a), int(b)) for a, b in zip(keys[0], ids[0])] == [(9, 3), (169, 2)]
    assert st["search_evals"] == 4
    ids, keys, st = g.search(q, 2, 1.3, 6, 5, 0, starts=[6, 5, 1])
    assert [(int(a), int(b)) for a, b in zip(keys[0], ids[0])] == [(169, 2), (529, 1)]
    assert st["search_evals"] == 6 and st["search_skipped"] == 0


@pytest.mark.parametrize("name,n0,speedup,kr", [("C0", 2000, 4.0, 10), ("C0", 2000, 1.0, 10), ("C1", 6000, 8.0, 10),
                                                ("C1", 6000, 3.0, 17), ("C2", 4000, 16.0, 20), ("C2", 4000, 2.0, 5)])
def test_search_matches_oracle(name, n0, speedup, kr):
    cfg = _cfg_small(name, n0=n0)
    X = D.initial_points(cfg)
    Q = D.query_points(cfg, 300)
    g = _graph(X, cfg.k)
    o = O.OracleGraph(cfg.metric, X, cfg.k)
    o.init_exact()
    gi, gk, gst = g.search(Q, kr, speedup, cfg.e_num, cfg.e_den, cfg.search_seed)
    oi, ok, ost = o.search(Q, kr, speedup, cfg.e_num, cfg.e_den, cfg.search_seed)
    _assert_rows_equal(cfg.metric, gi, gk, oi, ok, "search " + name)
    assert gst["search_evals"] == ost[:, 0].sum()
    assert gst["search_starts"] == ost[:, 1].sum()
    assert gst["search_skipped"] == ost[:, 2].sum()
    assert gst["search_expansions"] == ost[:, 3].sum()
    assert gst["search_evals"] == 300 * O.budget(n0, kr, speedup)


def test_search_expansion_infinite_and_one():
    cfg = _cfg_small("C1", n0=3000)
    X = D.initial_points(cfg)
    Q = D.query_points(cfg, 100)
    g = _graph(X, cfg.k)
    o = O.OracleGraph(cfg.metric, X, cfg.k)
    o.init_exact()
    for num, den in ((1, 0), (1, 1), (5, 1)):
        gi, gk, gst = g.search(Q, 10, 6.0, num, den, 7)
        oi, ok, ost = o.search(Q, 10, 6.0, num, den, 7)
        _assert_rows_equal(cfg.metric, gi, gk, oi, ok, "e=%d/%d" % (num, den))
        assert gst["search_skipped"] == ost[:, 2].sum()


# ---------------------------------------------------------------------------
# A1-A7 graph_insert_batch
# ---------------------------------------------------------------------------
def _run_stream(cfg, batches, nthreads=None):
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.n_insert)
    cap = cfg.n0 + cfg.n_insert + 8
    g = _graph(X, cfg.k, cap)
    o = O.OracleGraph(cfg.metric, X, cfg.k, capacity=cap)
    o.init_exact()
    pos = 0
    for B in batches:
        first, gst = g.insert_batch(S[pos:pos + B], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
        ost = o.insert_batch(S[pos:pos + B], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed,
                             nthreads)
        assert first == cfg.n0 + pos
        assert gst["search_evals"] == ost[:, 0].sum()
        assert gst["ball_nodes"] == ost[:, 4].sum()
        assert gst["proposals"] == ost[:, 5].sum()
        pos += B
        gi, gk = g.rows()
        oi, ok = o.rows()
        _assert_rows_equal(cfg.metric, gi, gk, oi, ok, "%s after %d inserts" % (cfg.name, pos))
    return g, o


def test_insert_C0_sequential_batches_of_one():
    cfg = _cfg_small("C0", n_insert=60)
    _run_stream(cfg, [1] * 60)


@pytest.mark.parametrize("keytable", [True, False])
@pytest.mark.parametrize("name,n0,depth,k", [("C2", 3000, 3, 20), ("C4", 1500, 2, 10), ("C1", 2500, 1, 1),
                                              ("C0", 400, 4, 32)])
def test_insert_batches_of_one_fast_path(name, n0, depth, k, keytable, monkeypatch):
    """B = 1 takes the fused launch (search + the insert's update by one warp; on small graphs with the
    key table); every metric, depths 1-4, k = 1..32: equal to the oracle after every insert, and the
    batched path (KNNG_NO_B1) reaches the same graph."""
    if not keytable:
        monkeypatch.setenv("KNNG_NO_KT", "1")
    cfg = _cfg_small(name, n0=n0, n_insert=40)
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.n_insert)
    cap = cfg.n0 + cfg.n_insert + 8
    g = _graph(X, k, cap)
    o = O.OracleGraph(cfg.metric, X, k, capacity=cap)
    o.init_exact()
    for i in range(cfg.n_insert):
        first, gst = g.insert_batch(S[i:i + 1], cfg.speedup, cfg.e_num, cfg.e_den, depth, cfg.search_seed)
        ost = o.insert_batch(S[i:i + 1], cfg.speedup, cfg.e_num, cfg.e_den, depth, cfg.search_seed)
        assert first == cfg.n0 + i and gst["kernel_launches"] <= 3
        assert gst["search_evals"] == ost[:, 0].sum() and gst["ball_nodes"] == ost[:, 4].sum()
        assert gst["proposals"] == ost[:, 5].sum()
        if i % 8 == 7 or i == cfg.n_insert - 1:
            gi, gk = g.rows()
            oi, ok = o.rows()
            _assert_rows_equal(cfg.metric, gi, gk, oi, ok, "%s B=1 after %d" % (name, i + 1))
    monkeypatch.setenv("KNNG_NO_B1", "1")
    h = _graph(X, k, cap)
    for i in range(cfg.n_insert):
        h.insert_batch(S[i:i + 1], cfg.speedup, cfg.e_num, cfg.e_den, depth, cfg.search_seed)
    hi, hk = h.rows()
    gi, gk = g.rows()
    assert (hi == gi).all() and (hk == gk).all()


@pytest.mark.parametrize("name,n0,part,env", [("C0", 2000, False, None), ("C1", 12000, False, None),
                                              ("C2", 3000, False, None), ("C4", 1500, False, None),
                                              ("C0", 2000, False, "KNNG_NO_KT"), ("C2", 3000, False, "KNNG_ESMEM"),
                                              ("C3", 6000, True, None), ("C4", 1500, True, None)])
def test_insert_sequential_matches_oracle(name, n0, part, env, monkeypatch):
    """graph_insert_sequential: n points one after another (one launch when unpartitioned: key table /
    gathers / global E words; a loop of B = 1 inserts when partitioned) == the oracle's n B = 1 inserts,
    rows and summed counters."""
    if env:
        monkeypatch.setenv(env, "1" if env != "KNNG_ESMEM" else "0")
    cfg = _cfg_small(name, n0=n0, n_insert=70)
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.n_insert)
    cap = cfg.n0 + cfg.n_insert + 8
    g = _graph(X, cfg.k, cap)
    o = O.OracleGraph(cfg.metric, X, cfg.k, capacity=cap)
    o.init_exact()
    if part:
        gp, gm, _ = g.partition_kmedoids(cfg.P, cfg.imbalance, 3, cfg.part_seed)
        op, om, _ = o.partition_kmedoids(cfg.P, cfg.imbalance, 3, cfg.part_seed)
        assert (gp == op).all()
        o.set_partition(op, om)
    pos = 0
    for n in (1, 45, 24):
        first, gst = g.insert_sequential(S[pos:pos + n], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
        tot = np.zeros(6, np.int64)
        for i in range(pos, pos + n):
            tot += o.insert_batch(S[i:i + 1], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)[0, :6]
        assert first == cfg.n0 + pos
        assert (gst["search_evals"], gst["search_starts"], gst["search_skipped"], gst["search_expansions"],
                gst["ball_nodes"], gst["proposals"]) == tuple(int(x) for x in tot), (name, n, gst, tot)
        pos += n
        gi, gk = g.rows()
        oi, ok = o.rows()
        _assert_rows_equal(cfg.metric, gi, gk, oi, ok, "%s sequential after %d" % (name, pos))


def test_insert_C1_shape():
    cfg = _cfg_small("C1", n0=20000, n_insert=2100)
    _run_stream(cfg, [1024, 1024, 52])


def test_insert_C2_shape_f32_depth3():
    cfg = _cfg_small("C2", n0=12000, n_insert=1100)
    _run_stream(cfg, [512, 512, 76])


def test_insert_edge_cases():
    # batch larger than the graph, k=1, depth 1, ragged dims, B=0
    rng = np.random.default_rng(3)
    for metric, dim, k, depth in ((O.U8, 3, 1, 1), (O.U8, 40, 4, 3), (O.F32, 7, 3, 2)):
        X = (rng.integers(0, 9, size=(40, dim)).astype(np.uint8) if metric == O.U8
             else rng.standard_normal((40, dim)).astype(np.float32))
        S = (rng.integers(0, 9, size=(120, dim)).astype(np.uint8) if metric == O.U8
             else rng.standard_normal((120, dim)).astype(np.float32))
        g = _graph(X, k, 200)
        o = O.OracleGraph(metric, X, k, capacity=200)
        o.init_exact()
        for lo, hi in ((0, 0), (0, 100), (100, 101), (101, 120)):
            g.insert_batch(S[lo:hi], 2.0, 6, 5, depth, 11)
            o.insert_batch(S[lo:hi], 2.0, 6, 5, depth, 11)
            gi, gk = g.rows()
            oi, ok = o.rows()
            _assert_rows_equal(metric, gi, gk, oi, ok, "edge m=%d d=%d k=%d" % (metric, dim, k))


def test_insert_errors():
    from paper_1602_06819_b200 import KnngGraph, KnngError
    g = KnngGraph(np.zeros((20, 4), np.uint8), 3, capacity=25)
    with pytest.raises(KnngError) as e:
        g.insert_batch(np.zeros((6, 4), np.uint8), 2.0, 6, 5, 2, 1)
    assert e.value.code == -8
    with pytest.raises(KnngError) as e:
        g.insert_batch(np.zeros((2, 5), np.uint8), 2.0, 6, 5, 2, 1)
    assert e.value.code == -1
    with pytest.raises(KnngError) as e:
        g.insert_batch(np.zeros((2, 4), np.uint8), 0.5, 6, 5, 2, 1)
    assert e.value.code == -1
    with pytest.raises(KnngError) as e:
        g.insert_batch(np.zeros((2, 4), np.uint8), 2.0, 6, 5, 0, 1)
    assert e.value.code == -1


# ---------------------------------------------------------------------------
# Full C1 size, in the launch configuration bench.py times (B = 1024): sampled outputs
# ---------------------------------------------------------------------------
def test_C1_full_size_sampled():
    cfg = D.CONFIGS["C1"]
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.batch)
    g = _graph(X, cfg.k, cfg.n0 + cfg.n_insert)
    o = O.OracleGraph(cfg.metric, X, cfg.k)
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(cfg.n0, 300, replace=False))
    oi, ok = o.exact_rows(sample)
    gi, gk = g.rows()
    _assert_rows_equal(cfg.metric, gi[sample], gk[sample], oi, ok, "C1 init sample")
    first, st = g.insert_batch(S, cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
    assert st["search_evals"] == cfg.batch * O.budget(cfg.n0, cfg.k, cfg.speedup)
    gi, gk = g.rows()
    # every stored key is the oracle's key of that pair; rows sorted, distinct, no self-loops
    allp = np.concatenate([X, S])
    for v in list(sample[:100]) + list(range(cfg.n0, cfg.n0 + 100)):
        row = gi[v].tolist()
        assert v not in row and len(set(row)) == cfg.k
        for a in range(cfg.k):
            assert O.key(cfg.metric, allp[v], allp[row[a]]) == int(gk[v, a])
        for a in range(cfg.k - 1):
            assert O.precedes(cfg.metric, int(gk[v, a]), row[a], int(gk[v, a + 1]), row[a + 1])
    # new rows: top-k of (own search result, peers) => at least as close as the exact peers-only top-k
    for i in range(0, cfg.batch, 97):
        D_peers = sorted((O.key(cfg.metric, S[i], S[j]), cfg.n0 + j) for j in range(cfg.batch) if j != i)
        assert int(gk[cfg.n0 + i, -1]) <= D_peers[cfg.k - 1][0]


# ---------------------------------------------------------------------------
# A9 partition_kmedoids, A4 partitioned search (Alg. 3), A8 placement (Alg. 5)
# ---------------------------------------------------------------------------
def test_partition_w7_hand_trace():
    X = D.line_points([0, 1, 2, 3, 10, 11, 12, 13])
    g = _graph(X, 2, 16)
    part, med, cost = g.partition_kmedoids(2, 1.0, 10, 0, init_medoids=[1, 5])
    assert part.tolist() == [0, 0, 0, 0, 1, 1, 1, 1]
    assert med.tolist() == [1, 5] and cost.tolist() == [6]
    p2, m2 = g.partition()
    assert p2.tolist() == part.tolist() and m2.tolist() == [1, 5]


@pytest.mark.parametrize("name,n0,P,imb", [("C3", 3000, 2, 1.0), ("C3", 5000, 8, 1.05), ("C2", 4000, 4, 1.1),
                                           ("C3", 12000, 2, 1.05), ("C0", 2000, 8, 1.05)])
def test_partition_matches_oracle(name, n0, P, imb):
    cfg = _cfg_small(name, n0=n0)
    X = D.initial_points(cfg)
    g = _graph(X, cfg.k)
    o = O.OracleGraph(cfg.metric, X, cfg.k)
    o.init_exact()
    gp, gm, gc = g.partition_kmedoids(P, imb, 6, cfg.part_seed)
    op, om, oc = o.partition_kmedoids(P, imb, 6, cfg.part_seed)
    assert gm.tolist() == om.tolist() and gc.tolist() == oc.tolist()
    assert (gp == op).all()
    assert np.bincount(gp, minlength=P).max() <= math.ceil(n0 * imb / P)


def test_partitioned_search_and_stream_C3_shape():
    cfg = _cfg_small("C3", n0=20000, n_insert=2200)
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.n_insert)
    Q = D.query_points(cfg, 200)
    cap = cfg.n0 + cfg.n_insert + 8
    g = _graph(X, cfg.k, cap)
    o = O.OracleGraph(cfg.metric, X, cfg.k, capacity=cap)
    o.init_exact()
    gp, gm, _ = g.partition_kmedoids(cfg.P, cfg.imbalance, 4, cfg.part_seed)
    op, om, _ = o.partition_kmedoids(cfg.P, cfg.imbalance, 4, cfg.part_seed)
    assert (gp == op).all() and gm.tolist() == om.tolist()
    o.set_partition(op, om)
    gi, gk, gst = g.search(Q, cfg.k, cfg.speedup, cfg.e_num, cfg.e_den, cfg.search_seed)
    oi, ok, ost = o.search(Q, cfg.k, cfg.speedup, cfg.e_num, cfg.e_den, cfg.search_seed)
    _assert_rows_equal(cfg.metric, gi, gk, oi, ok, "partitioned search")
    assert gst["search_evals"] == ost[:, 0].sum() and gst["search_expansions"] == ost[:, 3].sum()
    pos = 0
    for B in (1024, 1024, 152):
        g.insert_batch(S[pos:pos + B], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
        o.insert_batch(S[pos:pos + B], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
        pos += B
        gi, gk = g.rows()
        oi, ok = o.rows()
        _assert_rows_equal(cfg.metric, gi, gk, oi, ok, "partitioned stream after %d" % pos)
        gpart, _ = g.partition()
        assert (gpart == o.part_of[:o.n]).all()


def test_partition_errors():
    from paper_1602_06819_b200 import KnngError
    g = _graph(np.random.default_rng(0).integers(0, 255, (100, 4)).astype(np.uint8), 3)
    with pytest.raises(KnngError):
        g.partition_kmedoids(0, 1.0, 3, 0)
    with pytest.raises(KnngError):
        g.partition_kmedoids(300, 1.0, 3, 0)
    with pytest.raises(KnngError):
        g.partition_kmedoids(4, 0.5, 3, 0)


# ---------------------------------------------------------------------------
# Jaccard token sets (C4 shape): exact cross-multiplied keys, bit-exact
# ---------------------------------------------------------------------------
def test_jaccard_init_search_stream_and_partition():
    cfg = _cfg_small("C4", n0=3000, n_insert=900)
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.n_insert)
    Q = D.query_points(cfg, 150)
    cap = cfg.n0 + cfg.n_insert + 8
    g = _graph(X, cfg.k, cap)
    o = O.OracleGraph(cfg.metric, X, cfg.k, capacity=cap)
    o.init_exact()
    gi, gk = g.rows()
    _assert_rows_equal(cfg.metric, gi, gk, o.ids[:cfg.n0], o.keys[:cfg.n0], "jaccard init")
    gi, gk, gst = g.search(Q, cfg.k, 4.0, cfg.e_num, cfg.e_den, cfg.search_seed)
    oi, ok, ost = o.search(Q, cfg.k, 4.0, cfg.e_num, cfg.e_den, cfg.search_seed)
    _assert_rows_equal(cfg.metric, gi, gk, oi, ok, "jaccard search")
    assert gst["search_evals"] == ost[:, 0].sum() and gst["search_skipped"] == ost[:, 2].sum()
    # unpartitioned batches, then partition and continue (Alg. 5 placement)
    g.insert_batch(S[:300], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
    o.insert_batch(S[:300], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
    gi, gk = g.rows()
    oi, ok = o.rows()
    _assert_rows_equal(cfg.metric, gi, gk, oi, ok, "jaccard stream")
    gp, gm, gc = g.partition_kmedoids(cfg.P, cfg.imbalance, 4, cfg.part_seed)
    op, om, oc = o.partition_kmedoids(cfg.P, cfg.imbalance, 4, cfg.part_seed)
    assert (gp == op).all() and gm.tolist() == om.tolist() and gc.tolist() == oc.tolist()
    o.set_partition(op, om)
    for lo, hi in ((300, 812), (812, 900)):
        g.insert_batch(S[lo:hi], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
        o.insert_batch(S[lo:hi], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
        gi, gk = g.rows()
        oi, ok = o.rows()
        _assert_rows_equal(cfg.metric, gi, gk, oi, ok, "jaccard partitioned stream")
    gpart, _ = g.partition()
    assert (gpart == o.part_of[:o.n]).all()


def test_jaccard_edge_sets():
    # identical sets (ties -> id), disjoint sets (key 0/u), single-token sets, a long set (> QMAX tokens)
    rng = np.random.default_rng(5)
    sets = [np.array([1, 2, 3], np.uint32)] * 6 + [np.array([100 + i], np.uint32) for i in range(10)]
    sets += [np.sort(rng.choice(5000, size=int(rng.integers(1, 40)), replace=False)).astype(np.uint32)
             for _ in range(80)]
    sets += [np.arange(0, 900, 2, dtype=np.uint32), np.arange(0, 600, 3, dtype=np.uint32)]
    g = _graph(sets, 4, 200)
    o = O.OracleGraph(O.JAC, sets, 4, capacity=200)
    o.init_exact()
    gi, gk = g.rows()
    _assert_rows_equal(O.JAC, gi, gk, o.ids[:len(sets)], o.keys[:len(sets)], "jaccard edge init")
    new = [np.arange(0, 700, 2, dtype=np.uint32), np.array([1, 2, 3], np.uint32), np.array([7], np.uint32)]
    g.insert_batch(new, 1.5, 6, 5, 2, 3)
    o.insert_batch(new, 1.5, 6, 5, 2, 3)
    gi, gk = g.rows()
    oi, ok = o.rows()
    _assert_rows_equal(O.JAC, gi, gk, oi, ok, "jaccard edge insert")


# ---------------------------------------------------------------------------
# Multi-GPU decomposition (Alg. 3 + Alg. 5 over G ranks), G ranks emulated on one GPU: every
# replica must equal the single-GPU graph (and the oracle) for G = 1, 2, 4, 8
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["C3", "C4"])
def test_multi_rank_stages_are_G_invariant(name):
    from paper_1602_06819_b200.dist import insert_batch_staged
    n0 = 6000 if name == "C3" else 2500
    cfg = _cfg_small(name, n0=n0, n_insert=700)
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.n_insert)
    cap = cfg.n0 + cfg.n_insert + 8
    ref = _graph(X, cfg.k, cap)
    ref.partition_kmedoids(cfg.P, cfg.imbalance, 3, cfg.part_seed)
    o = O.OracleGraph(cfg.metric, X, cfg.k, capacity=cap)
    o.init_exact()
    op, om, _ = o.partition_kmedoids(cfg.P, cfg.imbalance, 3, cfg.part_seed)
    o.set_partition(op, om)
    batches = [(0, 300), (300, 301), (301, 700)]
    for lo, hi in batches:
        ref.insert_batch(S[lo:hi], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
        o.insert_batch(S[lo:hi], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
    ri, rk = ref.rows()
    oi, ok = o.rows()
    _assert_rows_equal(cfg.metric, ri, rk, oi, ok, "single-GPU reference")
    for G in (1, 2, 4, 8):
        reps = [_graph(X, cfg.k, cap) for _ in range(G)]
        for g in reps:
            g.partition_kmedoids(cfg.P, cfg.imbalance, 3, cfg.part_seed)
        for lo, hi in batches:
            insert_batch_staged(reps, list(range(G)), G, S[lo:hi], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth,
                                cfg.search_seed, cfg.P)
        for r, g in enumerate(reps):
            gi, gk = g.rows()
            _assert_rows_equal(cfg.metric, gi, gk, oi, ok, "G=%d rank %d" % (G, r))
            gpart, _ = g.partition()
            assert (gpart == o.part_of[:o.n]).all()
        for g in reps:
            g.close()


def test_query_sharded_unpartitioned_is_G_invariant():
    """Unpartitioned graphs (C1 shape): the batch's queries are sharded over G ranks;
    every replica equals the ORACLE's batch of the same points (and the single-GPU graph) for every G."""
    from paper_1602_06819_b200.dist import insert_batch_staged
    cfg = _cfg_small("C1", n0=5000, n_insert=1500)
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.n_insert)
    cap = cfg.n0 + cfg.n_insert + 8
    ref = _graph(X, cfg.k, cap)
    o = O.OracleGraph(cfg.metric, X, cfg.k, capacity=cap)
    o.init_exact()
    batches = [(0, 1024), (1024, 1025), (1025, 1500)]
    for lo, hi in batches:
        ref.insert_batch(S[lo:hi], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
        o.insert_batch(S[lo:hi], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
    ri, rk = o.rows()
    gi, gk = ref.rows()
    _assert_rows_equal(cfg.metric, gi, gk, ri, rk, "single-GPU vs oracle")
    for G in (2, 3, 8):
        reps = [_graph(X, cfg.k, cap) for _ in range(G)]
        for lo, hi in batches:
            insert_batch_staged(reps, list(range(G)), G, S[lo:hi], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth,
                                cfg.search_seed, 0)
        for r, g in enumerate(reps):
            gi, gk = g.rows()
            _assert_rows_equal(cfg.metric, gi, gk, ri, rk, "query-sharded G=%d rank %d" % (G, r))
        for g in reps:
            g.close()
