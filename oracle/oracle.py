"""Python driver for the CPU oracle (oracle/knng_oracle.c).  TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this module.  It shares nothing with
paper_1602_06819_b200/: it has its own C library, its own marshalling and
its own graph state held in numpy arrays.

Paper citations: P:n = line n of PAPER.md.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
import threading

import numpy as np

U8, F32, JAC, JW, COS = 0, 1, 2, 3, 4
CSR = (JAC, JW, COS)   # points held as uint32 sequences in CSR form (sets; strings of characters)
_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "knng_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()


def build(force=False):
    """Compile the oracle (plain C, -O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            P, i32, i64, u64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
            L.or_rng_hash.restype = u64
            L.or_rng_hash.argtypes = [u64, u64, u64, u64]
            L.or_rng_draw.restype = u64
            L.or_rng_draw.argtypes = [u64, u64, u64, u64, u64]
            L.or_rng_perm.restype = C.c_int64
            L.or_rng_perm.argtypes = [u64, u64, u64, u64, u64]
            L.or_budget.restype = i64
            L.or_budget.argtypes = [i64, i32, dbl]
            L.or_key.restype = C.c_uint32
            L.or_key.argtypes = [i32, i32, P, i64, P, i64]
            L.or_closer.argtypes = [i32, C.c_uint32, C.c_uint32]
            L.or_jw_fraction.argtypes = [C.c_uint32, C.POINTER(u64), C.POINTER(u64)]
            L.or_jw_fraction.restype = None
            L.or_precedes.argtypes = [i32, C.c_uint32, i64, C.c_uint32, i64]
            L.or_skip.argtypes = [i32, C.c_uint32, C.c_uint32, u64, u64]
            L.or_exact_rows.restype = None
            L.or_exact_rows.argtypes = [i32, i32, P, P, i64, i32, P, i64, P, P]
            L.or_ignns_search.restype = i64
            L.or_ignns_search.argtypes = [i32, i32, P, P, i64, P, i32, P, i64, P, i32,
                                          P, P, i64, i32, dbl, u64, u64, u64, i64, P, i64,
                                          P, P, P, i32]
            L.or_insert_batch.restype = i32
            L.or_insert_batch.argtypes = [i32, i32, P, P, i32, i64, P, P, i32, P, P, P, i64, P,
                                          i64, dbl, u64, u64, i32, u64, i32, P, i32]
            L.or_insert_sequential.restype = i32
            L.or_insert_sequential.argtypes = [i32, i32, P, P, i32, i64, P, P, dbl, u64, u64, i32,
                                               u64, P]
            L.or_graph_search.restype = i32
            L.or_graph_search.argtypes = [i32, i32, P, P, i32, i64, P, P, i32, P, P, P, i64,
                                          P, P, i64, i32, dbl, u64, u64, u64, i32, P, P, P, i32, P, i32]
            L.or_partition_kmedoids.restype = i32
            L.or_partition_kmedoids.argtypes = [i32, i32, P, P, i64, i32, P, i32, dbl, i32, u64,
                                                P, P, P, i64, i32, P]
            L.or_nearest_medoid.restype = i32
            L.or_nearest_medoid.argtypes = [i32, i32, P, P, P, i32, P, i64]
            L.or_stage_search.restype = i32
            L.or_stage_search.argtypes = [i32, i32, P, P, i32, i64, P, P, i32, P, P, P, i64, i64, i32, i32, dbl,
                                          u64, u64, u64, P, P, P]
            L.or_stage_ball.restype = i32
            L.or_stage_ball.argtypes = [i32, i32, P, P, i32, i64, P, P, P, i64, i64, i32, i64, P, P]
            L.or_stage_apply.restype = i32
            L.or_stage_apply.argtypes = [i32, i32, i64, P, P, i64, i64, P, P]
            _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def default_threads():
    return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# Keys.  U8: int32 squared L2; F32: fp32 bits (canonical order, reading Q24);
# JAC: (inter << 16) | union.
# ---------------------------------------------------------------------------
def key(metric, a, b):
    if metric in CSR:
        a = np.ascontiguousarray(a, np.uint32)
        b = np.ascontiguousarray(b, np.uint32)
        return int(lib().or_key(metric, 0, _p(a), len(a), _p(b), len(b)))
    dt = np.uint8 if metric == U8 else np.float32
    a = np.ascontiguousarray(a, dt)
    b = np.ascontiguousarray(b, dt)
    return int(lib().or_key(metric, a.shape[-1], _p(a), 0, _p(b), 0))


def key_value(metric, k):
    """Numeric view of a key: D for L2 metrics, similarity i/u for Jaccard, jw for Jaro-Winkler, cos^2 * |a|^2
    (dot^2 / |b|^2, the row-relative value) for the 2-gram cosine."""
    if metric == F32:
        return float(np.uint32(k).view(np.float32))
    if metric == JW:
        n, d = jw_fraction(k)
        return n / d
    if metric == COS:
        return (k >> 16) ** 2 / (k & 0xFFFF)
    if metric == JAC:
        i, u = k >> 16, k & 0xFFFF
        return i / u if u else 0.0
    return int(k)


def jw_fraction(key):
    """Jaro-Winkler value of a key as an exact fraction (numerator, denominator) (or_jw_fraction)."""
    L = lib()
    num, den = C.c_uint64(), C.c_uint64()
    L.or_jw_fraction(C.c_uint32(int(key)), C.byref(num), C.byref(den))
    return int(num.value), int(den.value)


def closer(metric, a, b):
    return bool(lib().or_closer(metric, a, b))


def precedes(metric, ka, ida, kb, idb):
    return bool(lib().or_precedes(metric, ka, ida, kb, idb))


def skip(metric, kr, kbest, e_num, e_den):
    return bool(lib().or_skip(metric, kr, kbest, e_num, e_den))


def rng_hash(seed, pid, part, draw):
    return int(lib().or_rng_hash(seed, pid, part, draw))


def rng_draw(seed, pid, part, draw, m):
    return int(lib().or_rng_draw(seed, pid, part, draw, m))


def rng_perm(seed, pid, part, j, m):
    """Restart draw j of a search over a pool of m nodes (Q4: a pseudo-random permutation; -1 past m)."""
    return int(lib().or_rng_perm(seed, pid, part, j, m))


def budget(m, k, speedup):
    return int(lib().or_budget(m, k, speedup))


# ---------------------------------------------------------------------------
# Paper formulas (pure closed forms)
# ---------------------------------------------------------------------------
def eager_speedup_model(k, d):
    """Table 1 / P:83-87: e_h = k/2^d, e_l = k - k/2^d, e_s = e_l/(1+e_h), speedup = k/e_s."""
    e_h = k / 2.0 ** d
    e_l = k - k / 2.0 ** d
    e_s = e_l / (1.0 + e_h)
    return e_h, e_l, e_s, k / e_s


def quality_factor(n, n_a, k, e_c):
    """e_m = n_a k + n k n_a/(n_a+n), e_u = (n+n_a)k - e_m, Q = (e_c-e_u)/e_m."""
    e_m = n_a * k + n * k * n_a / (n_a + n)
    e_u = (n + n_a) * k - e_m
    return e_m, e_u, (e_c - e_u) / e_m


def recall(result_ids, truth_ids):
    """Reading Q31: |result n truth| / k per query (mean over rows)."""
    result_ids = np.asarray(result_ids)
    truth_ids = np.asarray(truth_ids)
    k = truth_ids.shape[-1]
    hits = [len(set(r.tolist()) & set(t.tolist())) for r, t in zip(result_ids, truth_ids)]
    return float(np.mean(hits)) / k


def correct_edges(ids, exact_ids):
    """Number of (node, neighbour) pairs of the exact graph present in the graph."""
    return int(sum(len(set(a.tolist()) & set(b.tolist())) for a, b in zip(ids, exact_ids)))


# ---------------------------------------------------------------------------
# Oracle graph: state in numpy arrays, every step in the C oracle.
# ---------------------------------------------------------------------------
class OracleGraph:
    def __init__(self, metric, points, k, capacity=None, dim=None):
        self.metric = metric
        self.k = int(k)
        if metric in CSR:
            sets = list(points)
            n = len(sets)
            self.n = n
            self.cap = int(capacity or 2 * n)
            total = sum(len(s) for s in sets)
            self.tok = np.zeros(max(total * (self.cap // max(n, 1) + 1), 16), np.uint32)
            self.off = np.zeros(self.cap + 1, np.uint64)
            pos = 0
            for i, s in enumerate(sets):
                self.tok[pos:pos + len(s)] = s
                pos += len(s)
                self.off[i + 1] = pos
            self.dim = 0
            self.data = self.tok
        else:
            points = np.asarray(points)
            n, d = points.shape
            self.n = n
            self.cap = int(capacity or 2 * n)
            self.dim = d
            dt = np.uint8 if metric == U8 else np.float32
            self.data = np.zeros((self.cap, d), dt)
            self.data[:n] = points
            self.off = None
        self.ids = np.full((self.cap, self.k), -1, np.int32)
        self.keys = np.zeros((self.cap, self.k), np.uint32)
        self.P = 0
        self.part_of = None
        self.members = None
        self.member_cnt = None
        self.member_cap = 0
        self.medoids = None

    # -- store ----------------------------------------------------------
    def _append_points(self, pts):
        B = len(pts)
        if self.n + B > self.cap:
            raise RuntimeError("capacity exceeded")
        if self.metric in CSR:
            pos = int(self.off[self.n])
            need = pos + sum(len(s) for s in pts)
            if need > len(self.tok):
                self.tok = np.concatenate([self.tok, np.zeros(need - len(self.tok) + len(self.tok) // 2, np.uint32)])
                self.data = self.tok
            for i, s in enumerate(pts):
                self.tok[pos:pos + len(s)] = s
                pos += len(s)
                self.off[self.n + i + 1] = pos
        else:
            self.data[self.n:self.n + B] = np.asarray(pts)

    def point(self, i):
        if self.metric in CSR:
            return self.tok[int(self.off[i]):int(self.off[i + 1])]
        return self.data[i]

    # -- A0: exact rows -----------------------------------------------------
    def exact_rows(self, rows, nthreads=None, n=None):
        """Exact rows (AL1) for the given node ids over nodes 0..n-1."""
        n = self.n if n is None else n
        rows = np.ascontiguousarray(rows, np.int64)
        out_i = np.zeros((len(rows), self.k), np.int32)
        out_k = np.zeros((len(rows), self.k), np.uint32)
        nthreads = nthreads or default_threads()
        chunks = np.array_split(np.arange(len(rows)), max(1, min(nthreads, len(rows))))
        L = lib()

        def work(ix):
            if len(ix) == 0:
                return
            r = np.ascontiguousarray(rows[ix])
            oi = np.zeros((len(ix), self.k), np.int32)
            ok = np.zeros((len(ix), self.k), np.uint32)
            L.or_exact_rows(self.metric, self.dim, _p(self.data), _p(self.off), n, self.k,
                            _p(r), len(r), _p(oi), _p(ok))
            out_i[ix] = oi
            out_k[ix] = ok

        ths = [threading.Thread(target=work, args=(c,)) for c in chunks]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return out_i, out_k

    def init_exact(self, nthreads=None):
        ids, keys = self.exact_rows(np.arange(self.n), nthreads)
        self.ids[:self.n] = ids
        self.keys[:self.n] = keys

    def set_rows(self, ids, keys):
        self.ids[:self.n] = ids
        self.keys[:self.n] = keys

    # -- partitions (C3/C4) -------------------------------------------------------
    def set_partition(self, part_of, medoids):
        P = len(medoids)
        self.P = P
        self.part_of = np.zeros(self.cap, np.uint8)
        self.part_of[:self.n] = part_of
        self.member_cap = self.cap
        self.members = np.full((P, self.member_cap), -1, np.int32)
        self.member_cnt = np.zeros(P, np.int64)
        for p in range(P):
            m = np.nonzero(part_of[:self.n] == p)[0].astype(np.int32)
            self.members[p, :len(m)] = m
            self.member_cnt[p] = len(m)
        self.medoids = np.ascontiguousarray(medoids, np.int32)

    def partition_kmedoids(self, P, imbalance, max_iter, seed, init_medoids=None,
                           exact_limit=4096, ncand=64):
        part = np.zeros(self.n, np.uint8)
        med = np.zeros(P, np.int32)
        cost = np.full(max_iter + 1, -1, np.int64)
        im = None if init_medoids is None else np.ascontiguousarray(init_medoids, np.int32)
        rc = lib().or_partition_kmedoids(self.metric, self.dim, _p(self.data), _p(self.off), self.n,
                                         self.k, _p(self.ids), P, imbalance, max_iter, seed,
                                         _p(part), _p(med), _p(cost), exact_limit, ncand, _p(im))
        if rc < 0:
            raise RuntimeError("or_partition_kmedoids rc=%d" % rc)
        return part, med, cost[:rc]

    # -- A1..A8: one batch -------------------------------------------------------
    def insert_batch(self, pts, speedup, e_num, e_den, depth, seed, nthreads=None, route=0):
        """route=1: search only the nearest medoid's partition (reading Q18's routing variant)."""
        B = len(pts)
        n_t = self.n
        self._append_points(pts)
        st = np.zeros((B, 6), np.int64)
        rc = lib().or_insert_batch(self.metric, self.dim, _p(self.data), _p(self.off), self.k, n_t,
                                   _p(self.ids), _p(self.keys), self.P, _p(self.part_of),
                                   _p(self.members), _p(self.member_cnt), self.member_cap,
                                   _p(self.medoids), B, speedup, e_num, e_den, depth, seed,
                                   nthreads or default_threads(), _p(st), int(route))
        if rc:
            raise RuntimeError("or_insert_batch rc=%d" % rc)
        self.n = n_t + B
        return st

    def insert_sequential(self, pt, speedup, e_num, e_den, depth, seed):
        """Literal Alg. 1 + Alg. 2 for one point."""
        n_t = self.n
        self._append_points([pt] if self.metric in CSR else np.asarray(pt)[None])
        st = np.zeros(6, np.int64)
        rc = lib().or_insert_sequential(self.metric, self.dim, _p(self.data), _p(self.off), self.k,
                                        n_t, _p(self.ids), _p(self.keys), speedup, e_num, e_den,
                                        depth, seed, _p(st))
        if rc:
            raise RuntimeError("or_insert_sequential rc=%d" % rc)
        self.n = n_t + 1
        return st

    def search(self, queries, kr, speedup, e_num, e_den, seed, nthreads=None, full_scan=0, route=0):
        """graph_search; full_scan=1 with e_den=0 is the GNNS baseline; route=1 searches only the
        nearest medoid's partition (reading Q18's routing variant)."""
        if self.metric in CSR:
            qoff = np.zeros(len(queries) + 1, np.uint64)
            qoff[1:] = np.cumsum([len(q) for q in queries])
            qd = np.concatenate(queries).astype(np.uint32) if len(queries) else np.zeros(1, np.uint32)
        else:
            qd = np.ascontiguousarray(queries, self.data.dtype)
            qoff = None
        nq = len(queries)
        oi = np.zeros((nq, kr), np.int32)
        ok = np.zeros((nq, kr), np.uint32)
        st = np.zeros((nq, 4), np.int64)
        rc = lib().or_graph_search(self.metric, self.dim, _p(self.data), _p(self.off), self.k, self.n,
                                   _p(self.ids), _p(self.keys), self.P, _p(self.part_of),
                                   _p(self.members), _p(self.member_cnt), self.member_cap,
                                   _p(qd), _p(qoff), nq, kr, speedup, e_num, e_den, seed,
                                   nthreads or default_threads(), _p(oi), _p(ok), _p(st), int(full_scan),
                                   _p(self.medoids), int(route))
        if rc:
            raise RuntimeError("or_graph_search rc=%d" % rc)
        return oi, ok, st

    def ignns(self, q, kr, speedup, e_num, e_den, seed, pid, starts=None, part=0, pool=None, full_scan=0):
        """One iGNNS search on the current graph; optional injected starts.  full_scan=1:
        the GNNS baseline's walk (with e_den=0, no restart skipping: GNNS)."""
        if self.metric in CSR:
            qd = np.ascontiguousarray(q, np.uint32)
            qtok, qn, qdata = qd, len(qd), None
        else:
            qdata = np.ascontiguousarray(q, self.data.dtype)
            qtok, qn = None, 0
        if pool is None:
            m = self.n
            pool_a = None
        else:
            pool_a = np.ascontiguousarray(pool, np.int32)
            m = len(pool_a)
        st_a = None if starts is None else np.ascontiguousarray(starts, np.int32)
        oi = np.zeros(kr, np.int32)
        ok = np.zeros(kr, np.uint32)
        st = np.zeros(4, np.int64)
        part_of = self.part_of if pool is not None else None
        lib().or_ignns_search(self.metric, self.dim, _p(self.data), _p(self.off), self.n,
                              _p(self.ids), self.k, _p(pool_a), m, _p(part_of), part,
                              _p(qdata), _p(qtok), qn, kr, speedup, e_num, e_den, seed, pid,
                              _p(st_a), 0 if st_a is None else len(st_a), _p(oi), _p(ok), _p(st), int(full_scan))
        return oi, ok, dict(evals=int(st[0]), starts=int(st[1]), skipped=int(st[2]),
                            expansions=int(st[3]))

    def recompute_medoids(self, seed, epoch, exact_limit=4096, ncand=64):
        """Alg. 5's last step: the Alg. 4 update step on the current partition."""
        L = lib()
        if not hasattr(L, "_rm"):
            L.or_recompute_medoids.restype = C.c_int
            L.or_recompute_medoids.argtypes = [C.c_int64, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                               C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
            L._rm = True
        med = np.ascontiguousarray(self.medoids, np.int32).copy()
        cost = np.zeros(1, np.int64)
        L.or_recompute_medoids(self.n, self.k, _p(self.ids), self.P, _p(self.part_of), _p(med), seed, epoch,
                               exact_limit, ncand, _p(cost))
        self.medoids = med
        return med, int(cost[0])

    def nearest_medoid(self, x):
        if self.metric in CSR:
            xa = np.ascontiguousarray(x, np.uint32)
            nx = len(xa)
        else:
            xa = np.ascontiguousarray(x, self.data.dtype)
            nx = 0
        return int(lib().or_nearest_medoid(self.metric, self.dim, _p(self.data), _p(self.off),
                                           _p(self.medoids), self.P, _p(xa), nx))

    def rows(self):
        return self.ids[:self.n].copy(), self.keys[:self.n].copy()

    # -- the batch split the way a distributed run splits it (tests of the multi-GPU design) --
    def ball_bound(self, depth):
        b, pw = 0, 1
        for _ in range(depth):
            if b >= self.n:
                break
            pw *= self.k
            b += pw
        return min(b, self.n)

    def stage_search(self, pts, plo, phi, speedup, e_num, e_den, seed):
        """Ingest the batch (rows n..n+B-1, n unchanged) and search partitions [plo, phi)."""
        B = len(pts)
        self._append_points(pts)
        self.pend_B = B
        oi = np.full((B, phi - plo, self.k), -1, np.int32)
        ok = np.zeros((B, phi - plo, self.k), np.uint32)
        ev = np.zeros(1, np.int64)
        rc = lib().or_stage_search(self.metric, self.dim, _p(self.data), _p(self.off), self.k, self.n, _p(self.ids),
                                   _p(self.keys), self.P, _p(self.part_of), _p(self.members), _p(self.member_cnt),
                                   self.member_cap, B, plo, phi, speedup, e_num, e_den, seed, _p(oi), _p(ok), _p(ev))
        if rc:
            raise RuntimeError("or_stage_search rc=%d" % rc)
        return oi, ok

    def stage_update(self, C_ids, C_keys, qlo, qhi, depth, ballmax):
        """New rows of the whole batch (top-k of C_i and the peers, Q15), then the balls of
        queries [qlo, qhi) -> props [qhi-qlo][ballmax][2], counts."""
        import functools
        B, n_t, k = self.pend_B, self.n, self.k

        def cmp(a, b):
            return -1 if precedes(self.metric, a[0], a[1], b[0], b[1]) else 1
        for i in range(B):
            cand = [(int(C_keys[i, t]), int(C_ids[i, t])) for t in range(k) if C_ids[i, t] >= 0]
            cand += [(key(self.metric, self.point(n_t + i), self.point(n_t + j)), n_t + j) for j in range(B) if j != i]
            cand.sort(key=functools.cmp_to_key(cmp))
            cand = cand[:k] + [(0, -1)] * (k - len(cand[:k]))
            self.keys[n_t + i] = [c[0] for c in cand]
            self.ids[n_t + i] = [c[1] for c in cand]
        props = np.zeros((max(qhi - qlo, 0), ballmax, 2), np.int32)
        cnt = np.zeros(max(qhi - qlo, 0), np.int32)
        Ci = np.ascontiguousarray(C_ids, np.int32)
        rc = lib().or_stage_ball(self.metric, self.dim, _p(self.data), _p(self.off), k, n_t, _p(self.ids),
                                 _p(self.keys), _p(Ci), qlo, qhi, depth, ballmax, _p(props), _p(cnt))
        if rc:
            raise RuntimeError("or_stage_ball rc=%d" % rc)
        return props, cnt

    def stage_commit(self, props_all, cnt_all, ballmax):
        B, n_t = self.pend_B, self.n
        pa = np.ascontiguousarray(props_all, np.int32)
        ca = np.ascontiguousarray(cnt_all, np.int32)
        lib().or_stage_apply(self.metric, self.k, n_t, _p(self.ids), _p(self.keys), len(ca), ballmax, _p(pa), _p(ca))
        if self.P > 0:       # placement at the nearest medoid, batch order (Alg. 5)
            for i in range(B):
                p = self.nearest_medoid(self.point(n_t + i))
                self.part_of[n_t + i] = p
                self.members[p, self.member_cnt[p]] = n_t + i
                self.member_cnt[p] += 1
        self.n = n_t + B
        self.pend_B = 0


def merge_candidates(metric, cand_ids, cand_keys, world, P, k):
    """Alg. 3 'keep the k most similar' over rank-major gathered candidates [world][B][P/world][k]."""
    import functools
    ci = np.asarray(cand_ids).reshape(world, -1, P // world, k)
    ck = np.asarray(cand_keys).reshape(world, -1, P // world, k)
    B = ci.shape[1]
    out_i = np.full((B, k), -1, np.int32)
    out_k = np.zeros((B, k), np.uint32)

    def cmp(a, b):
        return -1 if precedes(metric, a[0], a[1], b[0], b[1]) else 1
    for b in range(B):
        c = sorted(((int(ck[r, b, j, t]), int(ci[r, b, j, t])) for r in range(world) for j in range(P // world)
                    for t in range(k) if ci[r, b, j, t] >= 0), key=functools.cmp_to_key(cmp))[:k]
        for t, (kk, ii) in enumerate(c):
            out_i[b, t], out_k[b, t] = ii, kk
    return out_i, out_k
