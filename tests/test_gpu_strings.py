"""GPU parity of the string measures (Jaro-Winkler; 2-gram cosine) through the
C ABI against the CPU oracle on the same seeded synthetic strings (datagen S1 / S2).  Integer keys:
bit-exact rows, keys and counters."""
import numpy as np
import pytest

import datagen as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu

NAMES = ["S1", "S2"]


def _graph(X, k, metric, cap=None):
    from paper_1602_06819_b200 import KnngGraph
    return KnngGraph(X, k, device=0, capacity=cap or 2 * len(X), metric=metric)


def _eq(gi, gk, oi, ok, what):
    bad = np.nonzero((gi != oi).any(1) | (gk != ok).any(1))[0]
    assert len(bad) == 0, "%s: %d rows differ, first %s: gpu %s %s oracle %s %s" % (
        what, len(bad), bad[:5], gi[bad[0]], gk[bad[0]], oi[bad[0]], ok[bad[0]])


@pytest.mark.parametrize("name", NAMES)
def test_string_init_search_and_stream(name):
    cfg = D.CONFIGS[name].with_sizes(n0=2500, n_insert=700)
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.n_insert)
    Q = D.query_points(cfg, 200)
    cap = cfg.n0 + cfg.n_insert + 8
    g = _graph(X, cfg.k, cfg.metric, cap)
    o = O.OracleGraph(cfg.metric, X, cfg.k, capacity=cap)
    o.init_exact()
    gi, gk = g.rows()
    _eq(gi, gk, o.ids[:cfg.n0], o.keys[:cfg.n0], name + " init")
    for sp, num, den, kr, fs in ((4.0, 6, 5, 10, 0), (1.0, 6, 5, 7, 0), (8.0, 1, 0, 12, 0), (4.0, 1, 0, 10, 1)):
        gi, gk, gst = g.search(Q, kr, sp, num, den, cfg.search_seed, full_scan=fs)
        oi, ok, ost = o.search(Q, kr, sp, num, den, cfg.search_seed, full_scan=fs)
        _eq(gi, gk, oi, ok, "%s search speedup %s e %d/%d kr %d gnns %d" % (name, sp, num, den, kr, fs))
        assert (gst["search_evals"], gst["search_starts"], gst["search_skipped"], gst["search_expansions"]) == \
            tuple(int(x) for x in ost.sum(0))
    pos = 0
    for B in (256, 256, 1, 187):
        first, gst = g.insert_batch(S[pos:pos + B], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
        ost = o.insert_batch(S[pos:pos + B], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
        assert first == cfg.n0 + pos
        assert gst["search_evals"] == ost[:, 0].sum() and gst["ball_nodes"] == ost[:, 4].sum()
        assert gst["proposals"] == ost[:, 5].sum()
        pos += B
        gi, gk = g.rows()
        oi, ok = o.rows()
        _eq(gi, gk, oi, ok, "%s after %d inserts" % (name, pos))


@pytest.mark.parametrize("env", [None, "KNNG_NO_KT"])
@pytest.mark.parametrize("name", NAMES)
def test_string_sequential_inserts(name, env, monkeypatch):
    """graph_insert_sequential (the paper's sequential algorithm, one launch; key table on small pools or
    gathers) == the oracle's B = 1 inserts; the update's keys are the row owners' (directed for COS)."""
    if env:
        monkeypatch.setenv(env, "1")
    cfg = D.CONFIGS[name].with_sizes(n0=1500, n_insert=60)
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.n_insert)
    cap = cfg.n0 + cfg.n_insert + 8
    g = _graph(X, cfg.k, cfg.metric, cap)
    o = O.OracleGraph(cfg.metric, X, cfg.k, capacity=cap)
    o.init_exact()
    pos = 0
    for n in (1, 35, 24):
        first, gst = g.insert_sequential(S[pos:pos + n], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth,
                                         cfg.search_seed)
        tot = np.zeros(6, np.int64)
        for i in range(pos, pos + n):
            tot += o.insert_batch(S[i:i + 1], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)[0, :6]
        assert (gst["search_evals"], gst["search_starts"], gst["search_skipped"], gst["search_expansions"],
                gst["ball_nodes"], gst["proposals"]) == tuple(int(x) for x in tot)
        pos += n
        gi, gk = g.rows()
        oi, ok = o.rows()
        _eq(gi, gk, oi, ok, "%s sequential after %d" % (name, pos))
    # batches of one through graph_insert_batch (the fused B = 1 launch) reach the same graph
    h = _graph(X, cfg.k, cfg.metric, cap)
    for i in range(cfg.n_insert):
        h.insert_batch(S[i:i + 1], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
    hi, hk = h.rows()
    gi, gk = g.rows()
    assert (hi == gi).all() and (hk == gk).all()


def test_string_edge_cases_and_errors():
    from paper_1602_06819_b200 import KnngError, KNNG_JARO_WINKLER, KNNG_COSINE_2GRAM, Strings, TokenSets
    rng = np.random.default_rng(3)
    # empty strings, one-character strings (zero 2-gram vector), duplicates (ties -> id), max length 127
    pts = [np.zeros(0, np.uint32), np.array([97], np.uint32), np.array([97], np.uint32)]
    pts += [rng.integers(97, 100, size=int(L)).astype(np.uint32) for L in rng.integers(0, 128, size=300)]
    pts += [np.full(127, 98, np.uint32), np.full(127, 98, np.uint32)]
    for metric, om in ((KNNG_JARO_WINKLER, O.JW), (KNNG_COSINE_2GRAM, O.COS)):
        g = _graph(pts, 8, metric)
        o = O.OracleGraph(om, pts, 8)
        o.init_exact()
        gi, gk = g.rows()
        _eq(gi, gk, o.ids[:len(pts)], o.keys[:len(pts)], "edge strings %d" % metric)
        gi, gk, _ = g.search(pts[:40], 8, 1.0, 6, 5, 3)
        oi, ok, _ = o.search(pts[:40], 8, 1.0, 6, 5, 3)
        _eq(gi, gk, oi, ok, "edge strings search %d" % metric)
        with pytest.raises(KnngError):                      # strings: unpartitioned graphs only
            g.partition_kmedoids(2, 1.05, 3, 1)
        with pytest.raises(KnngError):                      # > 127 characters
            g.insert_batch(Strings.from_list([np.full(128, 97, np.uint32)], metric), 4.0, 6, 5, 2, 1)
        with pytest.raises(KnngError):                      # metric mismatch
            g.insert_batch(TokenSets.from_list([np.array([1, 2], np.uint32)]), 4.0, 6, 5, 2, 1)


@pytest.mark.parametrize("name", NAMES)
def test_string_full_size_prefix(name):
    """S1 / S2 at n0 = 100,000: the GPU's exact graph on a seeded 150-row sample == the oracle's brute force;
    the oracle then consumes the GPU graph and the first 1,024-insert batch is compared row by row."""
    cfg = D.CONFIGS[name]
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.batch)
    cap = cfg.n0 + cfg.batch + 8
    g = _graph(X, cfg.k, cfg.metric, cap)
    o = O.OracleGraph(cfg.metric, X, cfg.k, capacity=cap)
    gi, gk = g.rows()
    sample = np.random.default_rng(11).choice(cfg.n0, 150, replace=False)
    si, sk = o.exact_rows(sample)
    _eq(gi[sample], gk[sample], si, sk, name + " init sample")
    o.set_rows(gi, gk)
    first, gst = g.insert_batch(S, cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
    ost = o.insert_batch(S, cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
    assert gst["search_evals"] == ost[:, 0].sum() and gst["proposals"] == ost[:, 5].sum()
    gi, gk = g.rows()
    oi, ok = o.rows()
    _eq(gi, gk, oi, ok, name + " first batch at full size")


@pytest.mark.parametrize("name", ["C4", "S2"])
def test_sequential_inserts_across_store_growth(name):
    """A long graph_insert_sequential on a CSR store (sets / strings): the ingest grows (moves) the token
    buffer, and the fused launch's update must read the moved store (regression: a stale view)."""
    cfg = D.CONFIGS[name].with_sizes(n0=1200, n_insert=160)
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.n_insert)
    cap = cfg.n0 + cfg.n_insert + 8
    g = _graph(X, cfg.k, cfg.metric, cap)
    o = O.OracleGraph(cfg.metric, X, cfg.k, capacity=cap)
    o.init_exact()
    first, gst = g.insert_sequential(S, cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)
    tot = np.zeros(6, np.int64)
    for i in range(cfg.n_insert):
        tot += o.insert_batch(S[i:i + 1], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed)[0, :6]
    assert gst["proposals"] == tot[5] and gst["ball_nodes"] == tot[4] and gst["search_evals"] == tot[0]
    gi, gk = g.rows()
    oi, ok = o.rows()
    _eq(gi, gk, oi, ok, name + " long sequential")
