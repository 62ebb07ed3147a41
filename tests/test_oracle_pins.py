"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a number the paper prints
(tests/golden/, cited), a closed form, a hand-worked example (SURVEY.md C.5,
re-derived by brute force here), a special case that reduces to brute
force, or an invariant the paper states.
"""
import itertools
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O
from tests import pyref as R
from datagen import line_points

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    for ln in open(os.path.join(GOLD, name)):
        ln = ln.strip()
        if ln and not ln.startswith("#"):
            rows.append([float(x) for x in ln.split()])
    return rows


# ---------------------------------------------------------------------------
# independent brute force (numpy / python; shares nothing with the C oracle)
# ---------------------------------------------------------------------------
def brute_key_u8(a, b):
    d = a.astype(np.int64) - b.astype(np.int64)
    return int((d * d).sum())


def brute_sim_jac(a, b):
    a, b = set(int(x) for x in a), set(int(x) for x in b)
    return Fraction(len(a & b), len(a | b))


def brute_rows_u8(X, k):
    X = X.astype(np.int64)
    D = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
    n = len(X)
    rows = []
    for v in range(n):
        cand = sorted((int(D[v, u]), u) for u in range(n) if u != v)
        rows.append(cand[:k])
    return rows


def brute_rows_jac(sets, k):
    n = len(sets)
    rows = []
    for v in range(n):
        cand = sorted(((-brute_sim_jac(sets[v], sets[u]), u) for u in range(n) if u != v))
        rows.append([(-s, u) for s, u in cand[:k]])
    return rows


def jac_key_sim(key):
    return Fraction(key >> 16, key & 0xFFFF)


def random_sets(rng, n, vocab=30, lo=2, hi=8):
    return [np.sort(rng.choice(vocab, size=rng.integers(lo, hi + 1), replace=False)).astype(np.uint32)
            for _ in range(n)]


# ---------------------------------------------------------------------------
# Table 1 and Q (numbers the paper prints / its formulas)
# ---------------------------------------------------------------------------
def test_table1_eager_model_matches_paper():
    for k, d, e_h, e_l, e_s, sp in _golden("table1_eager_speedup.txt"):
        m = O.eager_speedup_model(int(k), int(d))
        assert abs(m[0] - e_h) < 1e-12 and abs(m[1] - e_l) < 1e-12
        assert abs(m[2] - e_s) <= 0.01 and abs(m[3] - sp) <= 0.01


def test_quality_factor_formulas():
    for n, na, k, ec, em, eu, q in _golden("quality_factor.txt"):
        r = O.quality_factor(n, na, k, ec)
        assert math.isclose(r[0], em, rel_tol=1e-9)
        assert math.isclose(r[1], eu, rel_tol=1e-9, abs_tol=1e-9)
        assert math.isclose(r[2], q, rel_tol=1e-9, abs_tol=1e-12)


def test_quality_factor_identities_random():
    rng = np.random.default_rng(5)
    for _ in range(100):
        n, na, k = (int(x) for x in rng.integers(1, 10000, 3))
        ec = float(rng.integers(0, (n + na) * k + 1))
        em, eu, q = O.quality_factor(n, na, k, ec)
        assert math.isclose(em + eu, (n + na) * k, rel_tol=1e-12)
        assert math.isclose(q * em + eu, ec, rel_tol=1e-9, abs_tol=1e-6)


def test_recall_counts():
    assert O.recall([[1, 2, 3]], [[1, 2, 3]]) == 1.0
    assert O.recall([[4, 5, 6]], [[1, 2, 3]]) == 0.0
    assert O.recall([list(range(10))], [list(range(3, 13))]) == 0.7


# ---------------------------------------------------------------------------
# Metrics (closed forms)
# ---------------------------------------------------------------------------
def test_u8_key_closed_form():
    a = np.array([0, 0, 0], np.uint8)
    b = np.array([1, 2, 2], np.uint8)
    assert O.key(O.U8, a, b) == 9
    rng = np.random.default_rng(1)
    for d in (1, 3, 32, 128, 200):
        for _ in range(20):
            x = rng.integers(0, 256, d).astype(np.uint8)
            y = rng.integers(0, 256, d).astype(np.uint8)
            assert O.key(O.U8, x, y) == brute_key_u8(x, y)
    x = np.zeros(128, np.uint8)
    y = np.full(128, 255, np.uint8)
    assert O.key(O.U8, x, y) == 128 * 255 * 255  # maximum, 8,323,200 fits int32


def test_f32_canonical_key_within_fp64_bound():
    rng = np.random.default_rng(2)
    for d in (1, 5, 96, 128, 131, 300):
        for _ in range(20):
            x = rng.standard_normal(d).astype(np.float32)
            y = (x + 0.1 * rng.standard_normal(d)).astype(np.float32)
            exact = float(((x.astype(np.float64) - y.astype(np.float64)) ** 2).sum())
            got = O.key_value(O.F32, O.key(O.F32, x, y))
            # error bound ~ (3 + terms_per_lane + 5) * 2^-24 relative (Q24)
            assert abs(got - exact) <= 2e-6 * exact + 1e-30
    z = np.array([1.0, 2.0, 3.0], np.float32)
    assert O.key_value(O.F32, O.key(O.F32, z, z)) == 0.0
    assert O.key_value(O.F32, O.key(O.F32, np.zeros(3, np.float32), np.array([1, 2, 2], np.float32))) == 9.0


def test_jaccard_key_and_order():
    A = np.array([1, 2, 3, 4], np.uint32)
    B = np.array([3, 4, 5], np.uint32)
    Cc = np.array([1, 2], np.uint32)
    kab, kac = O.key(O.JAC, A, B), O.key(O.JAC, A, Cc)
    assert (kab >> 16, kab & 0xFFFF) == (2, 5)
    assert (kac >> 16, kac & 0xFFFF) == (2, 4)
    assert O.closer(O.JAC, kac, kab) and not O.closer(O.JAC, kab, kac)   # 2/4 > 2/5
    # 1/2 vs 2/4: equal similarity -> smaller id first
    k12, k24 = (1 << 16) | 2, (2 << 16) | 4
    assert not O.closer(O.JAC, k12, k24) and not O.closer(O.JAC, k24, k12)
    assert O.precedes(O.JAC, k24, 3, k12, 7) and not O.precedes(O.JAC, k12, 7, k24, 3)
    rng = np.random.default_rng(3)
    sets = random_sets(rng, 40)
    for a, b in itertools.combinations(sets[:15], 2):
        assert jac_key_sim(O.key(O.JAC, a, b)) == brute_sim_jac(a, b)


def test_skip_rule_boundaries():
    # W6 (U8, e = 6/5, D_best = 9): skip iff 5 (1+D_r) > 60
    assert not O.skip(O.U8, 11, 9, 6, 5)
    assert O.skip(O.U8, 12, 9, 6, 5)
    # equality never skips (strict rule); e = 1 skips exactly the worse ones
    assert not O.skip(O.U8, 9, 9, 1, 1) and O.skip(O.U8, 10, 9, 1, 1)
    # e = +inf (den = 0) never skips
    assert not O.skip(O.U8, 10 ** 6, 0, 1, 0)
    # W5 (Jaccard, e = 6/5): best 1/2, candidate 2/5: 0.4 < 0.4167 -> skip
    assert O.skip(O.JAC, (2 << 16) | 5, (1 << 16) | 2, 6, 5)
    assert not O.skip(O.JAC, (5 << 16) | 12, (1 << 16) | 2, 6, 5)   # 5/12 = 0.41667 = (1/2)/(6/5)
    # F32 follows the same rule as U8 on real D
    f = lambda x: int(np.float32(x).view(np.uint32))
    assert not O.skip(O.F32, f(11.0), f(9.0), 6, 5) and O.skip(O.F32, f(11.5), f(9.0), 6, 5)
    # the rule against similarities directly: s_r < s_max / e with s = 1/(1+D)
    rng = np.random.default_rng(4)
    for _ in range(2000):
        dr, db = (int(x) for x in rng.integers(0, 500, 2))
        num, den = (int(x) for x in rng.integers(1, 20, 2))
        if num < den:
            num, den = den, num
        want = Fraction(1, 1 + dr) < Fraction(1, 1 + db) / Fraction(num, den)
        assert O.skip(O.U8, dr, db, num, den) == want


# ---------------------------------------------------------------------------
# RNG: known-answer vectors from an independent Python implementation (Q4)
# ---------------------------------------------------------------------------
M64 = (1 << 64) - 1
G = 0x9E3779B97F4A7C15


def _mix(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _py_hash(seed, pid, part, draw):
    h = _mix((seed + G) & M64)
    h = _mix(h ^ ((pid + 2 * G) & M64))
    h = _mix(h ^ ((part + 3 * G) & M64))
    return _mix(h ^ ((draw + 4 * G) & M64))


def test_rng_known_answers_python_reimplementation():
    # splitmix64 finaliser known answer: the first output of SplitMix64 seeded with 0
    # (state += golden; mix) is 0xE220A8397B1DCDAF (Steele, Lea, Flood 2014 reference stream)
    assert _mix(G) == 0xE220A8397B1DCDAF
    rng = np.random.default_rng(9)
    for _ in range(300):
        s, pid, part, dr = (int(x) for x in rng.integers(0, 2 ** 62, 4))
        m = int(rng.integers(1, 10 ** 7))
        h = _py_hash(s, pid, part, dr)
        assert O.rng_hash(s, pid, part, dr) == h
        assert O.rng_draw(s, pid, part, dr, m) == (h * m) >> 64


def test_rng_uniformity():
    m = 16
    counts = np.zeros(m)
    N = 32000
    for j in range(N):
        counts[O.rng_draw(2001, 12345, 0, j, m)] += 1
    chi2 = ((counts - N / m) ** 2 / (N / m)).sum()
    assert chi2 < 40  # 15 dof; p ~ 5e-4


def test_rng_perm_known_answers_python_reimplementation():
    """Restart draws (Q4, round 2): the oracle's Feistel permutation equals tests/pyref.py's
    independent implementation of DESIGN.md's statement, including m = 1, powers of two and their
    neighbours, and j >= m (-1)."""
    rng = np.random.default_rng(11)
    ms = [1, 2, 3, 4, 5, 7, 8, 9, 255, 256, 257, 4096, 4097, 62500, 1 << 20, 1050000, (1 << 31) - 1]
    for t in range(600):
        m = ms[t % len(ms)] if t < 200 else int(rng.integers(1, 1 << 31))
        s, pid = (int(x) for x in rng.integers(0, 2 ** 62, 2))
        part = int(rng.integers(0, 8))
        j = int(rng.integers(0, m + 3))
        assert O.rng_perm(s, pid, part, j, m) == R.rng_perm(s, pid, part, j, m)
    assert O.rng_perm(1, 2, 3, 5, 5) == -1 and O.rng_perm(1, 2, 3, 0, 1) == 0


@pytest.mark.parametrize("m", [1, 2, 3, 6, 64, 65, 127, 500, 549, 1000, 4097])
def test_rng_perm_is_a_permutation(m):
    """Every pool node is drawn exactly once in m draws (so a draw never repeats an earlier draw)."""
    for s, pid, part in ((2000, 0, 0), (2003, 12345, 7)):
        v = sorted(O.rng_perm(s, pid, part, j, m) for j in range(m))
        assert v == list(range(m))


def test_rng_perm_first_draw_uniform():
    """The first draw pi(0) over many searches (pids) is uniform over the pool."""
    m, N = 13, 26000
    counts = np.zeros(m)
    for pid in range(N):
        counts[O.rng_perm(2001, pid, 0, 0, m)] += 1
    chi2 = ((counts - N / m) ** 2 / (N / m)).sum()
    assert chi2 < 40  # 12 dof; p ~ 1e-4


# ---------------------------------------------------------------------------
# A0 exact rows
# ---------------------------------------------------------------------------
def test_exact_rows_line():
    g = O.OracleGraph(O.U8, line_points([0, 1, 2, 3, 4]), k=2)
    g.init_exact(1)
    assert set(g.ids[0].tolist()) == {1, 2}
    assert set(g.ids[2].tolist()) == {1, 3}


def test_exact_rows_vs_brute_u8_and_invariants():
    rng = np.random.default_rng(11)
    X = rng.integers(0, 6, size=(60, 3)).astype(np.uint8)    # many exact ties
    g = O.OracleGraph(O.U8, X, k=5)
    g.init_exact(2)
    br = brute_rows_u8(X, 5)
    for v in range(60):
        assert [(int(a), int(b)) for a, b in zip(g.keys[v], g.ids[v])] == br[v]
        assert v not in g.ids[v] and len(set(g.ids[v].tolist())) == 5


def test_exact_rows_vs_brute_jac():
    rng = np.random.default_rng(12)
    S = random_sets(rng, 40, vocab=12)
    g = O.OracleGraph(O.JAC, S, k=4)
    g.init_exact(2)
    br = brute_rows_jac(S, 4)
    for v in range(40):
        assert [(jac_key_sim(int(a)), int(b)) for a, b in zip(g.keys[v], g.ids[v])] == br[v]


def test_exact_rows_f32_vs_fp64():
    rng = np.random.default_rng(13)
    X = rng.standard_normal((80, 7)).astype(np.float32)
    g = O.OracleGraph(O.F32, X, k=6)
    g.init_exact(2)
    X64 = X.astype(np.float64)
    D = ((X64[:, None] - X64[None]) ** 2).sum(-1)
    for v in range(80):
        d = D[v].copy()
        d[v] = np.inf
        want = np.argsort(d, kind="stable")[:6]
        assert g.ids[v].tolist() == want.tolist()      # no near-ties at this size
        got = np.array([O.key_value(O.F32, int(x)) for x in g.keys[v]])
        assert np.allclose(got, d[want], rtol=2e-6)


# ---------------------------------------------------------------------------
# W3: iGNNS hand traces with injected starts
# ---------------------------------------------------------------------------
W3_POINTS = [0, 10, 20, 30, 40, 100, 110, 120]


def _w3_graph():
    g = O.OracleGraph(O.U8, line_points(W3_POINTS), k=2)
    g.init_exact(1)
    return g


def test_w3_rows_are_the_exact_graph():
    g = _w3_graph()
    want = {0: [(100, 1), (400, 2)], 1: [(100, 0), (100, 2)], 2: [(100, 1), (100, 3)],
            3: [(100, 2), (100, 4)], 4: [(100, 3), (400, 2)], 5: [(100, 6), (400, 7)],
            6: [(100, 5), (100, 7)], 7: [(100, 6), (400, 5)]}
    for v, r in want.items():
        assert [(int(a), int(b)) for a, b in zip(g.keys[v], g.ids[v])] == r


def test_w3a_exhausts_pool_equals_linear_search():
    g = _w3_graph()
    ids, keys, st = g.ignns(np.array([33], np.uint8), 2, speedup=0.8, e_num=6, e_den=5, seed=0,
                            pid=0, starts=[1, 6, 7, 5])
    # budget = max(min(2, 8), floor(8/0.8)) = 10 > 8 -> capped by pool exhaustion
    assert [(int(a), int(b)) for a, b in zip(keys, ids)] == [(9, 3), (49, 4)]
    assert st["evals"] == 8 and st["skipped"] == 3


def test_w3b_budget_stops_before_fifth_eval():
    g = _w3_graph()
    ids, keys, st = g.ignns(np.array([33], np.uint8), 2, speedup=2.0, e_num=6, e_den=5, seed=0,
                            pid=0, starts=[1, 6, 7, 5])
    assert [(int(a), int(b)) for a, b in zip(keys, ids)] == [(9, 3), (169, 2)]
    assert st["evals"] == 4


def test_w3c_free_redraw_and_accepted_restart():
    g = _w3_graph()
    ids, keys, st = g.ignns(np.array([33], np.uint8), 2, speedup=1.3, e_num=6, e_den=5, seed=0,
                            pid=0, starts=[6, 5, 1])
    assert [(int(a), int(b)) for a, b in zip(keys, ids)] == [(169, 2), (529, 1)]
    assert st["evals"] == 6 and st["skipped"] == 0


# ---------------------------------------------------------------------------
# Search special cases and invariants
# ---------------------------------------------------------------------------
def _random_graph(metric, n, k, seed, dim=4):
    rng = np.random.default_rng(seed)
    if metric == O.U8:
        X = rng.integers(0, 40, size=(n, dim)).astype(np.uint8)
    elif metric == O.F32:
        X = rng.standard_normal((n, dim)).astype(np.float32)
    else:
        X = random_sets(rng, n, vocab=25)
    g = O.OracleGraph(metric, X, k=k)
    g.init_exact(2)
    return g, rng


def _query(metric, rng, dim=4):
    if metric == O.U8:
        return rng.integers(0, 40, size=dim).astype(np.uint8)
    if metric == O.F32:
        return rng.standard_normal(dim).astype(np.float32)
    return random_sets(rng, 1, vocab=25)[0]


def _linear_search(g, q, kr):
    keys = [O.key(g.metric, q, g.point(u)) for u in range(g.n)]
    order = sorted(range(g.n), key=lambda u: (0, 0))  # placeholder, replaced below
    import functools

    def cmp(a, b):
        if O.precedes(g.metric, keys[a], a, keys[b], b):
            return -1
        return 1

    order = sorted(range(g.n), key=functools.cmp_to_key(cmp))
    return order[:kr]


@pytest.mark.parametrize("metric", [O.U8, O.F32, O.JAC])
def test_budget_at_least_pool_is_linear_search(metric):
    g, rng = _random_graph(metric, 70, 5, 21 + metric)
    for qi in range(15):
        q = _query(metric, rng)
        ids, keys, st = g.ignns(q, 5, speedup=1.0, e_num=6, e_den=5, seed=7, pid=qi)
        assert st["evals"] == g.n
        if metric == O.JAC:
            want = brute_topk_jac(g, q, 5)
            assert [jac_key_sim(int(x)) for x in keys] == [s for s, _ in want]
            assert ids.tolist() == [u for _, u in want]
        elif metric == O.U8:
            D = [(brute_key_u8(q, g.point(u)), u) for u in range(g.n)]
            assert [(int(a), int(b)) for a, b in zip(keys, ids)] == sorted(D)[:5]
        else:
            assert ids.tolist() == _linear_search(g, q, 5)


def brute_topk_jac(g, q, kr):
    c = sorted(((-brute_sim_jac(q, g.point(u)), u) for u in range(g.n)))
    return [(-s, u) for s, u in c[:kr]]


@pytest.mark.parametrize("metric", [O.U8, O.F32, O.JAC])
def test_search_budget_soundness_determinism(metric):
    g, rng = _random_graph(metric, 200, 6, 31 + metric)
    for qi in range(20):
        q = _query(metric, rng)
        sp = float(rng.choice([2.0, 3.0, 7.5, 20.0]))
        ids, keys, st = g.ignns(q, 6, speedup=sp, e_num=6, e_den=5, seed=3, pid=qi)
        b = O.budget(g.n, 6, sp)
        assert b == max(min(6, g.n), math.floor(g.n / sp))
        assert st["evals"] == b                     # RNG searches always spend the budget
        assert st["skipped"] <= st["starts"] <= st["evals"]
        for i_, k_ in zip(ids, keys):               # soundness
            assert O.key(metric, q, g.point(int(i_))) == int(k_)
        for a in range(5):                          # sorted by edge order, distinct
            assert O.precedes(metric, int(keys[a]), int(ids[a]), int(keys[a + 1]), int(ids[a + 1]))
        ids2, keys2, st2 = g.ignns(q, 6, speedup=sp, e_num=6, e_den=5, seed=3, pid=qi)
        assert (ids2 == ids).all() and st2 == st     # determinism


def test_expansion_inf_never_skips_and_e1_skips_more():
    g, rng = _random_graph(O.U8, 300, 6, 41)
    tot_inf = tot_1 = 0
    for qi in range(30):
        q = _query(O.U8, rng)
        _, _, a = g.ignns(q, 6, speedup=3.0, e_num=1, e_den=0, seed=1, pid=qi)
        _, _, b = g.ignns(q, 6, speedup=3.0, e_num=1, e_den=1, seed=1, pid=qi)
        assert a["skipped"] == 0
        tot_inf += a["skipped"]
        tot_1 += b["skipped"]
    assert tot_1 > 0


# ---------------------------------------------------------------------------
# W1, W2: online insert (Alg. 1 + 2), batched vs sequential
# ---------------------------------------------------------------------------
def _rows(g, nodes):
    return {v: [(int(a), int(b)) for a, b in zip(g.keys[v], g.ids[v])] for v in nodes}


def test_w1_single_insert_equals_exact_graph():
    g = O.OracleGraph(O.U8, line_points([0, 10, 20, 30, 40]), k=2, capacity=10)
    g.init_exact(1)
    st = g.insert_batch(line_points([22]), speedup=1.0, e_num=6, e_den=5, depth=2, seed=5)
    r = _rows(g, range(6))
    assert r[5] == [(4, 2), (64, 3)]
    assert r[2] == [(4, 5), (100, 1)]
    assert r[3] == [(64, 5), (100, 2)]
    assert r[1] == [(100, 0), (100, 2)]
    assert r[4] == [(100, 3), (324, 5)]
    assert r[0] == [(100, 1), (400, 2)]
    assert st[0, 0] == 5 and st[0, 4] == 4 and st[0, 5] == 3   # evals, ball {2,3,1,4}, 3 proposals
    ex = O.OracleGraph(O.U8, line_points([0, 10, 20, 30, 40, 22]), k=2)
    ex.init_exact(1)
    assert (ex.ids[:6] == g.ids[:6]).all() and (ex.keys[:6] == g.keys[:6]).all()


def test_w2_sequential_vs_batched():
    base = line_points([0, 10, 20, 30, 40])
    seq = O.OracleGraph(O.U8, base, k=2, capacity=10)
    seq.init_exact(1)
    seq.insert_sequential(np.array([22], np.uint8), 1.0, 6, 5, 2, 5)
    seq.insert_sequential(np.array([24], np.uint8), 1.0, 6, 5, 2, 5)
    r = _rows(seq, range(7))
    assert r[6] == [(4, 5), (16, 2)]
    assert r[5] == [(4, 2), (4, 6)]
    assert r[2] == [(4, 5), (16, 6)]
    assert r[3] == [(36, 6), (64, 5)]
    assert r[4] == [(100, 3), (324, 5)]          # node 4 is at depth 3 for id 6
    bat = O.OracleGraph(O.U8, base, k=2, capacity=10)
    bat.init_exact(1)
    bat.insert_batch(line_points([22, 24]), 1.0, 6, 5, 2, 5)
    r = _rows(bat, range(7))
    assert r[5] == [(4, 2), (4, 6)]
    assert r[6] == [(4, 5), (16, 2)]
    assert r[2] == [(4, 5), (16, 6)]
    assert r[3] == [(36, 6), (64, 5)]
    assert r[4] == [(100, 3), (256, 6)]
    assert r[0] == [(100, 1), (400, 2)] and r[1] == [(100, 0), (100, 2)]
    ex = O.OracleGraph(O.U8, line_points([0, 10, 20, 30, 40, 22, 24]), k=2)
    ex.init_exact(1)
    assert (ex.ids[:7] == bat.ids[:7]).all()


@pytest.mark.parametrize("metric,depth", [(O.U8, 1), (O.U8, 2), (O.U8, 3), (O.F32, 2), (O.JAC, 2)])
def test_batch_of_one_equals_literal_sequential(metric, depth):
    g1, rng = _random_graph(metric, 120, 4, 51 + depth + 7 * metric)
    g2, _ = _random_graph(metric, 120, 4, 51 + depth + 7 * metric)
    g1.cap = g2.cap = 240
    for t in range(40):
        x = _query(metric, rng)
        s1 = g1.insert_batch([x] if metric == O.JAC else x[None], 5.0, 6, 5, depth, 99)
        s2 = g2.insert_sequential(x, 5.0, 6, 5, depth, 99)
        assert (g1.ids[:g1.n] == g2.ids[:g2.n]).all() and (g1.keys[:g1.n] == g2.keys[:g2.n]).all()
        assert s1[0, 0] == s2[0]


def _check_graph_invariants(g):
    for v in range(g.n):
        row = g.ids[v].tolist()
        assert v not in row and len(set(row)) == g.k and min(row) >= 0 and max(row) < g.n
        for a in range(g.k - 1):
            assert O.precedes(g.metric, int(g.keys[v, a]), row[a], int(g.keys[v, a + 1]), row[a + 1])
        for a in range(g.k):
            assert O.key(g.metric, g.point(v), g.point(row[a])) == int(g.keys[v, a])


@pytest.mark.parametrize("metric", [O.U8, O.F32, O.JAC])
def test_batches_keep_invariants_and_monotone_quality(metric):
    g, rng = _random_graph(metric, 150, 5, 61 + metric)
    g.cap = 400
    for b in range(4):
        B = int(rng.integers(1, 30))
        pts = [_query(metric, rng) for _ in range(B)]
        if metric != O.JAC:
            pts = np.stack(pts)
        old_k = g.keys[:g.n, -1].copy()
        old_i = g.ids[:g.n, -1].copy()
        n_old = g.n
        g.insert_batch(pts, 4.0, 6, 5, 2, 17)
        for v in range(n_old):          # monotone edge quality
            assert not O.precedes(metric, int(old_k[v]), int(old_i[v]), int(g.keys[v, -1]), int(g.ids[v, -1])) \
                or (old_k[v] == g.keys[v, -1] and old_i[v] == g.ids[v, -1])
        _check_graph_invariants(g)


def test_update_equals_python_ball_semantics():
    """Alg. 2 re-derived in plain Python: with speedup 1 the new row is the exact
    top-k (linear search); every node within DEPTH-1 out-hops of the new row over the
    pre-insert rows ends with top-k(old row + new point); every other row is unchanged.
    (SPEC's stronger 1-D claim does not hold in general: a mutual-nearest pair
    that no out-edge reaches never sees the new point, which the paper's Alg. 2 shares.)"""
    for seed in range(6):
        rng = np.random.default_rng(100 + seed)
        vals = rng.integers(0, 256, size=(70, 2)).astype(np.uint8)
        k, depth = 3, 1 + seed % 3
        g = O.OracleGraph(O.U8, vals[:20], k=k, capacity=80)
        g.init_exact(1)
        for x in vals[20:]:
            old_i, old_k = g.ids[:g.n].copy(), g.keys[:g.n].copy()
            n_t = g.n
            g.insert_batch(x[None], 1.0, 6, 5, depth, seed)
            D = [brute_key_u8(x, vals[u]) for u in range(n_t)]
            want_new = sorted((D[u], u) for u in range(n_t))[:k]
            assert [(int(a), int(b)) for a, b in zip(g.keys[n_t], g.ids[n_t])] == want_new
            ball, frontier = set(u for _, u in want_new), [u for _, u in want_new]
            for _ in range(depth - 1):
                nxt = []
                for v in frontier:
                    for u in old_i[v]:
                        if int(u) not in ball:
                            ball.add(int(u))
                            nxt.append(int(u))
                frontier = nxt
            for v in range(n_t):
                old = [(int(a), int(b)) for a, b in zip(old_k[v], old_i[v])]
                want = sorted(old + [(D[v], n_t)])[:k] if v in ball else old
                assert [(int(a), int(b)) for a, b in zip(g.keys[v], g.ids[v])] == want


# ---------------------------------------------------------------------------
# Partitioner (Alg. 4) and partitioned search (Alg. 3) / placement (Alg. 5)
# ---------------------------------------------------------------------------
W7_POINTS = [0, 1, 2, 3, 10, 11, 12, 13]


def test_w7_partitioner_hand_trace():
    g = O.OracleGraph(O.U8, line_points(W7_POINTS), k=2, capacity=16)
    g.init_exact(1)
    rows = _rows(g, range(8))
    assert rows[3] == [(1, 2), (4, 1)] and rows[7] == [(1, 6), (4, 5)]
    part, med, cost = g.partition_kmedoids(2, 1.0, 10, 0, init_medoids=[1, 5])
    assert part.tolist() == [0, 0, 0, 0, 1, 1, 1, 1]
    assert med.tolist() == [1, 5]
    assert cost.tolist() == [6]
    g.set_partition(part, med)
    assert g.nearest_medoid(np.array([9], np.uint8)) == 1      # D = 64 vs 4
    assert g.nearest_medoid(np.array([1], np.uint8)) == 0      # equal to medoid 0's point
    assert g.nearest_medoid(np.array([6], np.uint8)) == 0      # tie 25 vs 25 -> lowest p


def test_path_medoid_is_centre():
    # a-b-c path: 1-D points 0, 10, 20 with k=1 give edges 0->1, 1->0 (tie by id), 2->1
    g = O.OracleGraph(O.U8, line_points([0, 10, 20]), k=1, capacity=4)
    g.init_exact(1)
    part, med, cost = g.partition_kmedoids(1, 1.0, 3, 0)
    assert med.tolist() == [1] and cost[0] == 2


def _brute_hops(members, ids):
    ms = set(members)
    adj = {u: set() for u in members}
    for u in members:
        for v in ids[u]:
            if int(v) in ms:
                adj[u].add(int(v))
                adj[int(v)].add(u)
    best = None
    for c in sorted(members):
        dist = {c: 0}
        fr = [c]
        while fr:
            nf = []
            for u in fr:
                for w in adj[u]:
                    if w not in dist:
                        dist[w] = dist[u] + 1
                        nf.append(w)
            fr = nf
        s = sum(dist.get(u, len(members)) for u in members)
        if best is None or s < best[0]:
            best = (s, c)
    return best


@pytest.mark.parametrize("metric", [O.U8, O.JAC])
def test_partitioner_balance_cost_and_bruteforce_medoids(metric):
    g, rng = _random_graph(metric, 240, 4, 71 + metric)
    for P, imb in ((2, 1.0), (4, 1.1), (8, 1.05)):
        part, med, cost = g.partition_kmedoids(P, imb, 6, 5 + P)
        cap = math.ceil(240 * imb / P)
        sizes = np.bincount(part, minlength=P)
        assert sizes.max() <= cap and sizes.sum() == 240
        assert all(cost[i + 1] <= cost[i] for i in range(len(cost) - 1))
        tot = 0
        for p in range(P):
            mem = np.nonzero(part == p)[0].tolist()
            s, c = _brute_hops(mem, g.ids)
            assert med[p] == c
            tot += s
        assert tot == cost[-1]


def test_balance_spec_example():
    rng = np.random.default_rng(81)
    X = rng.integers(0, 256, size=(2000, 3)).astype(np.uint8)
    g = O.OracleGraph(O.U8, X, k=5)
    g.init_exact()
    for s in range(3):
        part, med, cost = g.partition_kmedoids(8, 1.1, 2, s)
        assert np.bincount(part, minlength=8).max() <= 275   # ceil(2000*1.1/8)


@pytest.mark.parametrize("metric", [O.U8, O.JAC])
def test_partitioned_search_special_cases(metric):
    g, rng = _random_graph(metric, 160, 5, 91 + metric)
    part, med, _ = g.partition_kmedoids(4, 1.05, 3, 2)
    g.set_partition(part, med)
    qs = [_query(metric, rng) for _ in range(10)]
    qa = qs if metric == O.JAC else np.stack(qs)
    # speedup 1: every partition exhausted -> exact linear search over all nodes
    ids, keys, st = g.search(qa, 5, 1.0, 6, 5, 3)
    for i, q in enumerate(qs):
        if metric == O.U8:
            D = sorted((brute_key_u8(q, g.point(u)), u) for u in range(g.n))[:5]
            assert [(int(a), int(b)) for a, b in zip(keys[i], ids[i])] == D
        else:
            assert [(jac_key_sim(int(a)), int(b)) for a, b in zip(keys[i], ids[i])] == brute_topk_jac(g, q, 5)
    # P = 1 partitioned == unpartitioned
    h, _ = _random_graph(metric, 160, 5, 91 + metric)
    u_ids, u_keys, u_st = h.search(qa, 5, 6.0, 6, 5, 3)
    h.set_partition(np.zeros(160, np.uint8), np.array([0], np.int32))
    p_ids, p_keys, p_st = h.search(qa, 5, 6.0, 6, 5, 3)
    assert (u_ids == p_ids).all() and (u_st == p_st).all()


def test_partitioned_insert_places_and_keeps_invariants():
    g, rng = _random_graph(O.U8, 200, 5, 101)
    g.cap = 400
    part, med, _ = g.partition_kmedoids(4, 1.05, 3, 2)
    g.set_partition(part, med)
    pts = np.stack([_query(O.U8, rng) for _ in range(25)])
    n_t = g.n
    g.insert_batch(pts, 4.0, 6, 5, 2, 8)
    for i in range(25):
        p = g.nearest_medoid(pts[i])
        assert g.part_of[n_t + i] == p
        assert n_t + i in g.members[p, :g.member_cnt[p]].tolist()
    for p in range(4):
        m = g.members[p, :g.member_cnt[p]]
        assert (np.diff(m) > 0).all()
    assert g.member_cnt.sum() == g.n
    _check_graph_invariants(g)
