"""Pins of the oracle's string measures (P:289 Jaro-Winkler, P:292 cosine of 2-gram
count vectors) against things other than the oracle itself (CPU only):
  * the textbook values of tests/golden/string_measures.txt (cited there);
  * tests/pyref.py's exact-fraction re-derivations (Python lists / Counters, no shared code);
  * invariants SPEC states (symmetry, range, Winkler boost >= Jaro);
  * the search / update special cases that hold for every metric (budget >= pool is linear search,
    a batch of one is the literal sequential Alg. 1 + 2).
"""
import functools
import os
from fractions import Fraction

import numpy as np
import pytest

import datagen as D
from oracle import oracle as O

from . import pyref as R

GOLD = os.path.join(os.path.dirname(__file__), "golden", "string_measures.txt")


def _s(x):
    return np.asarray([ord(c) for c in x], np.uint32)


def _jw_value(a, b):
    n, d = O.jw_fraction(O.key(O.JW, a, b))
    return Fraction(n, d)


def _cos_sq(a, b):
    """cos^2 from the oracle's directed keys: dot and |b|^2 from key(a -> b), |a|^2 from key(b -> a)."""
    kab, kba = O.key(O.COS, a, b), O.key(O.COS, b, a)
    dot = kab >> 16
    assert dot == kba >> 16                      # the inner product is symmetric
    return Fraction(dot * dot, (kab & 0xFFFF) * (kba & 0xFFFF))


def _rand_strings(rng, n, lo=0, hi=14, alpha=4):
    return [rng.integers(97, 97 + alpha, size=int(rng.integers(lo, hi + 1))).astype(np.uint32) for _ in range(n)]


def test_golden_textbook_values():
    rows = [ln.split() for ln in open(GOLD) if ln.strip() and not ln.startswith("#")]
    assert len(rows) == 10
    for meas, a, b, v in rows:
        a, b = _s(a.replace("_", "")), _s(b.replace("_", ""))
        if meas == "jw":
            got = float(_jw_value(a, b))
        else:
            got = float(_cos_sq(a, b)) ** 0.5
        assert abs(got - float(v)) <= 5e-5, (meas, a, b, got, v)


def test_jw_textbook_fractions():
    # the worked examples' exact values (m, t, l in the golden file's comment)
    assert _jw_value(_s("MARTHA"), _s("MARHTA")) == Fraction(173, 180)
    assert _jw_value(_s("DWAYNE"), _s("DUANE")) == Fraction(21, 25)
    assert _jw_value(_s("DIXON"), _s("DICKSONX")) == Fraction(61, 75)


def test_jw_matches_python_rederivation_random():
    rng = np.random.default_rng(5)
    for alpha in (2, 3, 6, 26):
        A = _rand_strings(rng, 400, 0, 20, alpha)
        B = _rand_strings(rng, 400, 0, 20, alpha)
        for a, b in zip(A, B):
            assert _jw_value(a, b) == R.jaro_winkler(a.tolist(), b.tolist()), (a, b)


def test_cos_matches_python_rederivation_random():
    rng = np.random.default_rng(6)
    for alpha in (2, 3, 6):
        A = _rand_strings(rng, 400, 0, 25, alpha)
        B = _rand_strings(rng, 400, 0, 25, alpha)
        for a, b in zip(A, B):
            assert _cos_sq(a, b) == R.cosine_2gram_sq(a.tolist(), b.tolist()), (a, b)
            k = O.key(O.COS, a, b)
            nb = sum(v * v for v in R.bigram_counts(b.tolist()).values())
            assert k & 0xFFFF == max(nb, 1)


def test_invariants_symmetry_range_boost():
    rng = np.random.default_rng(7)
    A = _rand_strings(rng, 600, 0, 16, 3)
    B = _rand_strings(rng, 600, 0, 16, 3)
    for a, b in zip(A, B):
        jw_ab, jw_ba = _jw_value(a, b), _jw_value(b, a)
        assert jw_ab == jw_ba and 0 <= jw_ab <= 1
        # Winkler boost never lowers Jaro: jaro from the key with l := 0
        k = O.key(O.JW, a, b)
        n0, d0 = O.jw_fraction(k & ~(7 << 14))
        assert jw_ab >= Fraction(n0, d0)
        c = _cos_sq(a, b)
        assert c == _cos_sq(b, a) and 0 <= c <= 1
    assert _jw_value(_s("abcd"), _s("abcd")) == 1 and _cos_sq(_s("abab"), _s("abab")) == 1


@pytest.mark.parametrize("metric", [O.JW, O.COS])
def test_closer_and_skip_match_fractions(metric):
    """closer / the skip rule (s_r < s_max / e) on keys sharing an owner, against exact fractions."""
    rng = np.random.default_rng(8 + metric)
    val = (lambda a, b: R.jaro_winkler(a, b)) if metric == O.JW else (lambda a, b: R.cosine_2gram_sq(a, b))
    for _ in range(300):
        q = _rand_strings(rng, 1, 1, 16, 3)[0]
        x, y = _rand_strings(rng, 2, 0, 16, 3)
        kx, ky = O.key(metric, q, x), O.key(metric, q, y)
        vx, vy = val(q.tolist(), x.tolist()), val(q.tolist(), y.tolist())
        assert O.closer(metric, kx, ky) == (vx > vy)
        for num, den in ((6, 5), (1, 1), (5, 1), (7, 3)):
            e = Fraction(num, den)
            want = vx < vy / e if metric == O.JW else vx < vy / (e * e)   # COS values are squares
            assert O.skip(metric, kx, ky, num, den) == want
        assert not O.skip(metric, kx, ky, 1, 0)


def _brute_rows(metric, pts, k):
    val = R.jaro_winkler if metric == O.JW else R.cosine_2gram_sq
    rows = []
    for v in range(len(pts)):
        cand = [(-val(pts[v].tolist(), pts[u].tolist()), u) for u in range(len(pts)) if u != v]
        rows.append([u for _, u in sorted(cand)[:k]])
    return np.asarray(rows, np.int32)


@pytest.mark.parametrize("metric", [O.JW, O.COS])
def test_exact_rows_vs_python_brute_force(metric):
    rng = np.random.default_rng(9 + metric)
    pts = _rand_strings(rng, 70, 1, 12, 3)
    g = O.OracleGraph(metric, pts, k=6)
    g.init_exact(2)
    assert (g.ids[:70] == _brute_rows(metric, pts, 6)).all()


def _string_graph(metric, n, k, seed):
    rng = np.random.default_rng(seed)
    g = O.OracleGraph(metric, _rand_strings(rng, n, 1, 12, 4), k=k)
    g.init_exact(2)
    return g, rng


@pytest.mark.parametrize("metric", [O.JW, O.COS])
def test_budget_at_least_pool_is_linear_search(metric):
    g, rng = _string_graph(metric, 80, 5, 31 + metric)
    for qi in range(12):
        q = _rand_strings(rng, 1, 1, 12, 4)[0]
        ids, keys, st = g.ignns(q, 5, speedup=1.0, e_num=6, e_den=5, seed=7, pid=qi)
        assert st["evals"] == g.n
        val = R.jaro_winkler if metric == O.JW else R.cosine_2gram_sq
        want = [u for _, u in sorted((-val(q.tolist(), g.point(u).tolist()), u) for u in range(g.n))[:5]]
        assert ids.tolist() == want


@pytest.mark.parametrize("metric,depth", [(O.JW, 1), (O.JW, 2), (O.COS, 2), (O.COS, 3)])
def test_batch_of_one_equals_literal_sequential(metric, depth):
    g1, rng = _string_graph(metric, 120, 4, 41 + depth + 7 * metric)
    g2, _ = _string_graph(metric, 120, 4, 41 + depth + 7 * metric)
    for t in range(30):
        x = _rand_strings(rng, 1, 1, 12, 4)[0]
        s1 = g1.insert_batch([x], 5.0, 6, 5, depth, 99)
        s2 = g2.insert_sequential(x, 5.0, 6, 5, depth, 99)
        assert (g1.ids[:g1.n] == g2.ids[:g2.n]).all() and (g1.keys[:g1.n] == g2.keys[:g2.n]).all()
        assert s1[0, 0] == s2[0]


@pytest.mark.parametrize("metric", [O.JW, O.COS])
def test_rows_hold_their_owners_keys(metric):
    """After batches of inserts every row v holds key(v -> u) of each entry u (directed keys for COS),
    sorted by edge order, k distinct ids, no self-loop."""
    g, rng = _string_graph(metric, 150, 5, 61 + metric)
    g.cap = 400
    for b in range(3):
        g.insert_batch(_rand_strings(rng, int(rng.integers(1, 25)), 1, 12, 4), 4.0, 6, 5, 2, 17)
    for v in range(g.n):
        row = g.ids[v].tolist()
        assert v not in row and len(set(row)) == g.k
        for a in range(g.k - 1):
            assert O.precedes(metric, int(g.keys[v, a]), row[a], int(g.keys[v, a + 1]), row[a + 1])
        for a in range(g.k):
            assert O.key(metric, g.point(v), g.point(row[a])) == int(g.keys[v, a])


def test_datagen_string_recipe():
    for name in ("S1", "S2"):
        cfg = D.CONFIGS[name].with_sizes(n0=500)
        X = D.initial_points(cfg)
        assert len(X) == 500 and all(1 <= len(x) <= 127 for x in X)
        assert set(np.concatenate(X).tolist()) <= set(D.ALPHABET.tolist())
        assert all((a == b).all() for a, b in zip(D.stream_points(cfg, 0, 10), D.stream_points(cfg, 0, 20)[:10]))


def _jw_counts_a_side(a, b):
    """(m, T) of the textbook matching: a's characters in order take the first free equal b character."""
    w = max(max(len(a), len(b)) // 2 - 1, 0)
    used = [False] * len(b)
    amatch = []
    for i, c in enumerate(a):
        for j in range(max(0, i - w), min(len(b), i + w + 1)):
            if not used[j] and b[j] == c:
                used[j] = True
                amatch.append(i)
                break
    bmatch = [j for j in range(len(b)) if used[j]]
    return len(amatch), sum(a[i] != b[j] for i, j in zip(amatch, bmatch))


def _jw_counts_b_side_pointers(a, b):
    """(m, T) the way the GPU's table evaluator matches: b's characters in order, each consuming the next
    feasible position of the same character in a (per-character pointers; positions < j - w skipped)."""
    w = max(max(len(a), len(b)) // 2 - 1, 0)
    pos = {}
    for i, c in enumerate(a):
        pos.setdefault(c, []).append(i)
    ptr = {c: 0 for c in pos}
    amatch, bmatch = [], []
    for j, c in enumerate(b):
        if c not in pos:
            continue
        p, lst = ptr[c], pos[c]
        while p < len(lst) and lst[p] < j - w:
            p += 1
        if p < len(lst) and lst[p] <= j + w:
            amatch.append(lst[p])
            bmatch.append(j)
            p += 1
        ptr[c] = p
    amatch.sort()
    return len(amatch), sum(a[i] != b[j] for i, j in zip(amatch, bmatch))


def test_jw_matching_side_independent():
    """The GPU evaluates JW by scanning the candidate against the query's per-character position lists
    (matching from the candidate's side); pinned here: that matching has the textbook (m, T) on random
    strings of small alphabets (many repeated characters) and every length up to the 127-character bound."""
    rng = np.random.default_rng(12)
    for alpha, hi in ((2, 20), (3, 40), (5, 127), (26, 127)):
        for _ in range(1500 if hi <= 40 else 300):
            a = rng.integers(0, alpha, size=int(rng.integers(0, hi + 1))).tolist()
            b = rng.integers(0, alpha, size=int(rng.integers(0, hi + 1))).tolist()
            assert _jw_counts_b_side_pointers(a, b) == _jw_counts_a_side(a, b), (a, b)
            assert _jw_counts_b_side_pointers(b, a) == _jw_counts_a_side(a, b), (a, b)
