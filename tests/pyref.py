"""Plain-Python re-derivations of the paper's procedures, used ONLY as pins of the C oracle.

Nothing here imports oracle/ or the CUDA package: every function is written from the paper (and the
readings of DESIGN.md) in exact arithmetic -- Python ints and Fractions, no floating point in any
decision -- so that a dropped term, a wrong sign or a transposed operand in the oracle fails a test.

  * mulhi RNG (reading Q4): the SplitMix64 finaliser chain, restated from Steele, Lea & Flood (2014).
  * iGNNS (section 3) LITERALLY: no "restart when moving onto an expanded node" shortcut
    (reading Q9) -- a walk that reaches an expanded node re-scans its row on cached keys.
  * the GNNS baseline walk (section 2.2): all k neighbours evaluated, move to the best.
  * Alg. 4 with the sampled-candidate medoid update of reading Q22 and the
    acceptance rule of Q23, every score compared as an exact fraction.
  * the string measures of SURVEY 8(f)#4 (P:289 Jaro-Winkler, P:292 cosine of 2-gram count vectors) as
    exact fractions (the cosine as its square, which orders the same way).
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
U8, F32, JAC = 0, 1, 2


def mix64(z):
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def rng_hash(seed, pid, part, draw):
    h = mix64((seed + GOLDEN) & M64)
    h = mix64(h ^ ((pid + 2 * GOLDEN) & M64))
    h = mix64(h ^ ((part + 3 * GOLDEN) & M64))
    return mix64(h ^ ((draw + 4 * GOLDEN) & M64))


def rng_draw(seed, pid, part, draw, m):
    """index = floor(h * m / 2^64) (reading Q4)."""
    return (rng_hash(seed, pid, part, draw) * m) >> 64


def _lowbias32(z):
    for sh, mul in ((16, 0x7FEB352D), (15, 0x846CA68B)):
        z = ((z ^ (z >> sh)) * mul) % 2**32
    return z ^ (z >> 16)


def rng_perm(seed, pid, part, j, m):
    """Restart draw j of a search over m pool nodes (reading Q4, round 2): a 6-round Feistel permutation
    of the b-bit integers (b = max(6, bits of m - 1)), halves of b // 2 (high) and b - b // 2 (low) bits that
    swap widths every round, cycle-walked into [0, m).  Written from DESIGN.md's statement, not from
    the oracle's C."""
    if j >= m:
        return -1
    b = max(6, (m - 1).bit_length())
    h = mix64((seed + GOLDEN) & M64)
    h = mix64(h ^ ((pid + 2 * GOLDEN) & M64))
    pre = mix64(h ^ ((part + 3 * GOLDEN) & M64))
    keys = [((pre >> (16 * (i % 4))) % 2**32) ^ ((0x9E3779B9 * (i + 1)) % 2**32) for i in range(6)]
    widths = [b // 2, b - b // 2]           # [left, right]
    x = j
    while True:
        left, right = divmod(x, 2 ** widths[1])
        wl, wr = widths
        for key in keys:
            f = _lowbias32(right ^ key) % 2 ** wl
            left, right, wl, wr = right, left ^ f, wr, wl
        x = left * 2 ** wr + right
        if x < m:
            return x


# ---------------------------------------------------------------------------
# Exact metric values.  L2: D as an exact integer / Fraction (inputs are integer-valued, so the
# fp32 canonical sum of the oracle is exact too); Jaccard: (inter, union).
# ---------------------------------------------------------------------------
def metric_value(metric, a, b):
    if metric == JAC:
        sa, sb = set(int(x) for x in a), set(int(x) for x in b)
        i = len(sa & sb)
        return (i, len(sa) + len(sb) - i)
    d = [Fraction(float(x)) - Fraction(float(y)) for x, y in zip(a, b)]
    return sum(x * x for x in d)


def similarity(metric, v):
    """s = 1/(1+D) for L2 metrics (reading Q1), i/u for Jaccard."""
    if metric == JAC:
        i, u = v
        return Fraction(i, u) if u else Fraction(0)
    return Fraction(1) / (1 + v)


def closer(metric, a, b):
    """a strictly more similar than b (metric value only)."""
    return similarity(metric, a) > similarity(metric, b)


def sort_key(metric, v, node):
    """Edge order: more similar first, equal similarity -> smaller id."""
    return (-similarity(metric, v), node)


def packed_key(metric, v):
    """The library / oracle key format of a metric value."""
    if metric == JAC:
        return (v[0] << 16) | v[1]
    if metric == U8:
        return int(v)
    return int(np.float32(float(v)).view(np.uint32))


def skip(metric, v_r, v_best, e_num, e_den):
    """discard a restart r when s_r < s_max / e (strict), e = num/den, den = 0 -> never."""
    if e_den == 0:
        return False
    return similarity(metric, v_r) < similarity(metric, v_best) * Fraction(e_den, e_num)


def budget(m, kr, speedup):
    """P:89 + reading Q6: max(min(k, |pool|), floor(|pool| / speedup))."""
    return max(min(kr, m), math.floor(m / speedup))


# ---------------------------------------------------------------------------
# iGNNS, literally
# ---------------------------------------------------------------------------
def ignns_literal(metric, point, rows, q, kr, speedup, e_num, e_den, seed, pid, pool=None, part=0, starts=None,
                  full_scan=False):
    """Returns (ids, packed keys, stats) of the top-kr evaluated nodes.

    full_scan=True is the GNNS baseline's walk (section 2.2): the similarity of EVERY neighbour
    of the current node is computed and the walk moves to the most similar one (first in row order
    among equals) if it improves on the current node.

    point(i) -> the stored point i; rows[i] -> node i's neighbour ids (stored order, -1 padded);
    pool = sorted node ids of the searched partition (None: all nodes 0..len(rows)-1)."""
    pool = list(range(len(rows))) if pool is None else list(pool)
    inpool = set(pool)
    m = len(pool)
    b = budget(m, kr, speedup)
    val = {}                    # evaluated node -> metric value (the search cache)
    c = 0                       # similarities computed
    j = 0                       # draw counter
    st = dict(evals=0, starts=0, skipped=0)
    first = True

    def best():
        return min(val, key=lambda u: sort_key(metric, val[u], u))

    while True:
        if c == b or c == m:                       # budget; whole pool evaluated (Q7)
            break
        while True:                                # random restart; redraws are free (Q4)
            if starts is not None:
                if j >= len(starts):
                    return _finish(metric, val, kr, st, c)
                r = starts[j]
            else:
                r = pool[rng_perm(seed, pid, part, j, m)]
            j += 1
            if r not in val:
                break
        vb = val[best()] if val else None          # s_max before r
        val[r] = metric_value(metric, q, point(r))
        c += 1
        st["starts"] += 1
        if not first and vb is not None and skip(metric, val[r], vb, e_num, e_den):
            st["skipped"] += 1                     # the skipped start stays in the result (Q5)
            continue
        first = False
        cur = r
        while full_scan:                           # GNNS: best of all k neighbours
            nb = None
            for v in rows[cur]:
                v = int(v)
                if v < 0 or v not in inpool:
                    continue
                if v not in val:
                    if c == b:
                        return _finish(metric, val, kr, st, c)
                    val[v] = metric_value(metric, q, point(v))
                    c += 1
                if closer(metric, val[v], val[cur]) and (nb is None or closer(metric, val[v], val[nb])):
                    nb = v
            if nb is None:
                break
            cur = nb
        while not full_scan:                       # hill climbing, eager first improvement
            moved = False
            for v in rows[cur]:
                v = int(v)
                if v < 0 or v not in inpool:       # edges leaving the pool are skipped (Q10)
                    continue
                if v not in val:
                    if c == b:                     # the over-budget evaluation is not performed
                        return _finish(metric, val, kr, st, c)
                    val[v] = metric_value(metric, q, point(v))
                    c += 1
                if closer(metric, val[v], val[cur]):
                    cur = v
                    moved = True
                    break
            if not moved:                          # local maximum -> restart
                break
    return _finish(metric, val, kr, st, c)


def _finish(metric, val, kr, st, c):
    st["evals"] = c
    order = sorted(val, key=lambda u: sort_key(metric, val[u], u))[:kr]
    return [int(u) for u in order], [packed_key(metric, val[u]) for u in order], st


# ---------------------------------------------------------------------------
# Alg. 4: balanced k-medoids, readings Q21-Q23
# ---------------------------------------------------------------------------
def _hop_sum(c, members, adj):
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
    return sum(dist.get(u, len(members)) for u in members)


def _best_medoid(members, adj, cur, seed, tag, stream, exact_limit, ncand):
    """(hop sum, id) of the candidate minimising the hop sum; candidates: every member when
    |C| <= exact_limit, else (Q22) the current medoid and ncand - 1 draws of stream (seed, tag, stream, j)."""
    if len(members) <= exact_limit:
        cands = members
    else:
        cands = ([cur] if cur in set(members) else []) + [
            members[rng_draw(seed, tag, stream, j, len(members))] for j in range(ncand - 1)]
    return min((_hop_sum(c, members, adj), c) for c in cands)   # ties -> smaller id


def _cluster_adj(members, rows):
    ms = set(members)
    adj = {u: set() for u in members}
    for u in members:
        for v in rows[u]:
            v = int(v)
            if v in ms:
                adj[u].add(v)
                adj[v].add(u)
    return adj


def recompute_medoids(rows, part, med, seed, epoch, exact_limit=4096, ncand=64):
    """Alg. 5's last step: every medoid becomes its cluster's hop-sum minimiser on the current
    graph and partition (stream tag 0xFFFFFFFD, stream epoch * P + p).  Returns (medoids, total cost)."""
    P = len(med)
    out, cost = [], 0
    for p in range(P):
        members = [u for u in range(len(part)) if part[u] == p]
        if not members:
            out.append(int(med[p]))
            continue
        bs, bc = _best_medoid(members, _cluster_adj(members, rows), int(med[p]), seed, 0xFFFFFFFD, epoch * P + p,
                              exact_limit, ncand)
        out.append(bc)
        cost += bs
    return out, cost


def nearest_medoid(metric, point, q, med):
    """Placement / routing target: argmin_p D(q, medoid_p), ties -> lowest p."""
    best = None
    for p, m in enumerate(med):
        v = metric_value(metric, q, point(int(m)))
        if best is None or closer(metric, v, best[0]):
            best = (v, p)
    return best[1]


def kmedoids(metric, point, rows, P, imbalance, max_iter, seed, exact_limit=4096, ncand=64, init=None):
    """Returns (part, medoids, costs of the kept iterations)."""
    n = len(rows)
    cap = math.ceil(n * imbalance / P)
    if init is not None:
        med = [int(x) for x in init]
    else:
        med, jd = [], 0
        while len(med) < P:                        # P distinct seeded draws (Alg. 4 line 1)
            cnd = rng_draw(seed, 0xFFFFFFFF, 0, jd, n)
            jd += 1
            if cnd not in med:
                med.append(cnd)
    part_out, costs, prev = None, [], None
    for it in range(max_iter):
        # assign: ascending id, eligible clusters only, score s(m, u) * (1 - |C|/cap)
        size = [0] * P
        part = [0] * n
        for u in range(n):
            best, bscore = None, None
            for p in range(P):
                if size[p] >= cap:
                    continue
                sc = similarity(metric, metric_value(metric, point(u), point(med[p]))) * Fraction(cap - size[p], cap)
                if best is None or sc > bscore or (sc == bscore and (size[p], med[p]) < (size[best], med[best])):
                    best, bscore = p, sc
            part[u] = best
            size[best] += 1
        # update: member minimising the hop sum in the cluster-induced undirected view (Q29)
        newmed, cost = [], 0
        for p in range(P):
            members = [u for u in range(n) if part[u] == p]
            if not members:
                newmed.append(med[p])
                continue
            adj = _cluster_adj(members, rows)
            bs, bc = _best_medoid(members, adj, med[p], seed, 0xFFFFFFFE, it * P + p, exact_limit, ncand)
            newmed.append(bc)
            cost += bs
        if it > 0 and cost > prev:                 # Q23: an iteration that raises the cost is not kept
            break
        part_out = part
        costs.append(cost)
        prev = cost
        changed = newmed != med
        med = newmed
        if not changed:
            break
    return part_out, med, costs


# ---------------------------------------------------------------------------
# String measures, exact
# ---------------------------------------------------------------------------
def jaro_winkler(a, b):
    """Textbook Jaro-Winkler as a Fraction: Jaro (matching window max(|a|,|b|)//2 - 1, characters of a
    matched in order to the first unused equal character of b inside the window, t = half the matched
    characters out of order) plus the Winkler boost l/10 (1 - jaro), l = common prefix <= 4."""
    a, b = list(a), list(b)
    if not a or not b:
        return Fraction(0)
    w = max(max(len(a), len(b)) // 2 - 1, 0)
    used = [False] * len(b)
    a_seq = []
    for i, c in enumerate(a):
        for j in range(max(0, i - w), min(len(b), i + w + 1)):
            if not used[j] and b[j] == c:
                used[j] = True
                a_seq.append(c)
                break
    b_seq = [c for c, u in zip(b, used) if u]
    m = len(a_seq)
    if m == 0:
        return Fraction(0)
    t = Fraction(sum(x != y for x, y in zip(a_seq, b_seq)), 2)
    jaro = (Fraction(m, len(a)) + Fraction(m, len(b)) + (m - t) / m) / 3
    ell = 0
    while ell < min(4, len(a), len(b)) and a[ell] == b[ell]:
        ell += 1
    return jaro + Fraction(ell, 10) * (1 - jaro)


def bigram_counts(s):
    from collections import Counter
    s = list(s)
    return Counter(zip(s, s[1:]))


def cosine_2gram_sq(a, b):
    """cos^2 of the 2-gram count vectors as a Fraction (0 when either vector is zero)."""
    ca, cb = bigram_counts(a), bigram_counts(b)
    dot = sum(v * cb[g] for g, v in ca.items())
    na, nb = sum(v * v for v in ca.values()), sum(v * v for v in cb.values())
    if na == 0 or nb == 0:
        return Fraction(0)
    return Fraction(dot * dot, na * nb)

