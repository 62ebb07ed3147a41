"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic: it only draws points.
Both `oracle/` and `paper_1602_06819_b200/` consume its arrays; neither
imports the other.  Recipes follow BASELINE.json `configs` and SURVEY.md
section 8(d); readings Q26/Q27 fix what the configs leave open.

Every draw uses numpy's PCG64 keyed by (seed, purpose, chunk) so that any
prefix of a stream is identical whatever its total length:
    purpose 0: mixture means      purpose 1: initial points
    purpose 2: stream chunk c     (chunk = 4096 points)
    purpose 3: graph_search query sets
"""
from __future__ import annotations

import dataclasses
import numpy as np

CHUNK = 4096

U8, F32, JAC, JW, COS = 0, 1, 2, 3, 4
CSR = (JAC, JW, COS)   # points as lists of uint32 arrays (token sets; strings of characters)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    metric: int
    n0: int             # initial graph size
    dim: int            # vector dim (u8/f32), unused for JAC
    clusters: int
    sigma: float
    k: int
    n_insert: int
    batch: int
    speedup: float
    e_num: int          # expansion e = e_num / e_den   (Q2: 1.2 = 6/5)
    e_den: int
    depth: int
    P: int = 0          # 0 = unpartitioned
    imbalance: float = 1.05
    data_seed: int = 0
    search_seed: int = 0
    part_seed: int = 0

    def with_sizes(self, n0=None, n_insert=None, batch=None, **kw):
        d = dataclasses.asdict(self)
        if n0 is not None:
            d["n0"] = n0
        if n_insert is not None:
            d["n_insert"] = n_insert
        if batch is not None:
            d["batch"] = batch
        d.update(kw)
        return Config(**d)


def _cfg(c, **kw):
    return Config(data_seed=1000 + c, search_seed=2000 + c, part_seed=3000 + c, **kw)


# BASELINE.json configs[0..4]  (SURVEY.md 8(d) "Concrete inputs")
CONFIGS = {
    "C0": _cfg(0, name="C0", metric=U8, n0=2000, dim=32, clusters=8, sigma=12.0, k=10,
               n_insert=200, batch=1, speedup=4.0, e_num=6, e_den=5, depth=2),
    "C1": _cfg(1, name="C1", metric=U8, n0=100_000, dim=128, clusters=64, sigma=20.0, k=10,
               n_insert=10_000, batch=1024, speedup=8.0, e_num=6, e_den=5, depth=2),
    "C2": _cfg(2, name="C2", metric=F32, n0=1_000_000, dim=96, clusters=256, sigma=0.15, k=20,
               n_insert=100_000, batch=4096, speedup=16.0, e_num=6, e_den=5, depth=3),
    "C3": _cfg(3, name="C3", metric=U8, n0=8_000_000, dim=128, clusters=1024, sigma=20.0, k=10,
               n_insert=1_000_000, batch=8192, speedup=32.0, e_num=6, e_den=5, depth=2,
               P=8, imbalance=1.05),
    "C4": _cfg(4, name="C4", metric=JAC, n0=2_000_000, dim=0, clusters=0, sigma=0.0, k=10,
               n_insert=200_000, batch=4096, speedup=16.0, e_num=6, e_den=5, depth=2,
               P=8, imbalance=1.05),
}

# the paper's string workloads (P:289 SPAM subjects under Jaro-Winkler, P:292 Wikipedia
# pages under the 2-gram cosine) on synthetic strings (their corpora are absent): `clusters` templates,
# each point a template with random edits (STR_RECIPE).  Not BASELINE.json configs: parity / bench cases.
CONFIGS["S1"] = _cfg(5, name="S1", metric=JW, n0=100_000, dim=0, clusters=2000, sigma=0.0, k=10,
                     n_insert=10_000, batch=1024, speedup=8.0, e_num=6, e_den=5, depth=2)
CONFIGS["S2"] = _cfg(6, name="S2", metric=COS, n0=100_000, dim=0, clusters=2000, sigma=0.0, k=10,
                     n_insert=10_000, batch=1024, speedup=8.0, e_num=6, e_den=5, depth=2)


def _rng(seed, purpose, chunk=0):
    return np.random.Generator(np.random.PCG64([int(seed), int(purpose), int(chunk)]))


# ---------------------------------------------------------------------------
# Gaussian mixtures ("mixture of gaussian distributions"; Q27)
# ---------------------------------------------------------------------------
def _means(cfg: Config):
    r = _rng(cfg.data_seed, 0)
    if cfg.metric == U8:
        return r.uniform(32.0, 224.0, size=(cfg.clusters, cfg.dim))
    return r.standard_normal(size=(cfg.clusters, cfg.dim))


def _mixture(cfg: Config, means, r, n):
    lab = r.integers(0, cfg.clusters, size=n)
    x = means[lab] + cfg.sigma * r.standard_normal(size=(n, cfg.dim))
    if cfg.metric == U8:
        return np.clip(np.rint(x), 0, 255).astype(np.uint8)
    return x.astype(np.float32)


# ---------------------------------------------------------------------------
# Zipf token sets (Q26): L ~ U{5..50}; Zipf(1.1) ranks over 50,000 drawn until
# L distinct; token = rank - 1; sorted.
# ---------------------------------------------------------------------------
VOCAB = 50_000
ZIPF_S = 1.1
_ZIPF_CDF = None


def _zipf_cdf():
    global _ZIPF_CDF
    if _ZIPF_CDF is None:
        w = 1.0 / np.arange(1, VOCAB + 1, dtype=np.float64) ** ZIPF_S
        c = np.cumsum(w)
        _ZIPF_CDF = c / c[-1]
    return _ZIPF_CDF


def _token_sets(r, n):
    cdf = _zipf_cdf()
    lens = r.integers(5, 51, size=n)
    sets = []
    for L in lens:
        got = []
        seen = set()
        while len(got) < L:
            draws = np.searchsorted(cdf, r.random(2 * int(L)), side="right")
            for t in draws:
                t = int(min(t, VOCAB - 1))
                if t not in seen:
                    seen.add(t)
                    got.append(t)
                    if len(got) == L:
                        break
        sets.append(np.sort(np.asarray(got, dtype=np.uint32)))
    return sets


# ---------------------------------------------------------------------------
# Synthetic strings (8(f)#4): alphabet a-z and space (code points); template t of a config has length
# U{10..60} (JW, subject-like) or U{40..120} (COS, text-like) drawn from the alphabet; a point is a
# uniformly chosen template with each character substituted (p 0.08), deleted (p 0.04) or followed by an
# inserted character (p 0.04); lengths are clipped to 1..127 (the metrics' bound).
# ---------------------------------------------------------------------------
ALPHABET = np.array([ord(c) for c in "abcdefghijklmnopqrstuvwxyz "], dtype=np.uint32)
STR_RECIPE = dict(p_sub=0.08, p_del=0.04, p_ins=0.04, max_len=127)


def _templates(cfg: Config):
    r = _rng(cfg.data_seed, 0)
    lo, hi = (10, 61) if cfg.metric == JW else (40, 121)
    lens = r.integers(lo, hi, size=cfg.clusters)
    return [ALPHABET[r.integers(0, len(ALPHABET), size=int(L))] for L in lens]


def _strings(cfg: Config, tmpl, r, n):
    out = []
    lab = r.integers(0, len(tmpl), size=n)
    for t in lab:
        base = tmpl[int(t)]
        u = r.random((len(base), 3))
        subs = ALPHABET[r.integers(0, len(ALPHABET), size=len(base))]
        ins = ALPHABET[r.integers(0, len(ALPHABET), size=len(base))]
        s = []
        for i, ch in enumerate(base):
            if u[i, 1] < STR_RECIPE["p_del"]:
                continue
            s.append(int(subs[i]) if u[i, 0] < STR_RECIPE["p_sub"] else int(ch))
            if u[i, 2] < STR_RECIPE["p_ins"]:
                s.append(int(ins[i]))
        if not s:
            s = [int(base[0])]
        out.append(np.asarray(s[:STR_RECIPE["max_len"]], dtype=np.uint32))
    return out


def _csr_points(cfg: Config, r, n):
    return _token_sets(r, n) if cfg.metric == JAC else _strings(cfg, _templates(cfg), r, n)


def sets_to_csr(sets):
    off = np.zeros(len(sets) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(s) for s in sets])
    tok = np.concatenate(sets).astype(np.uint32) if sets else np.zeros(0, np.uint32)
    return off, tok


# ---------------------------------------------------------------------------
# Public API
# ---------------------------------------------------------------------------
def initial_points(cfg: Config):
    """u8/f32: array [n0, dim]; JAC: list of sorted uint32 arrays."""
    r = _rng(cfg.data_seed, 1)
    if cfg.metric in CSR:
        return _csr_points(cfg, r, cfg.n0)
    return _mixture(cfg, _means(cfg), r, cfg.n0)


def stream_points(cfg: Config, start: int, count: int):
    """Points start .. start+count-1 of the insert stream (prefix-stable)."""
    if count <= 0:
        if cfg.metric in CSR:
            return []
        dt = np.uint8 if cfg.metric == U8 else np.float32
        return np.zeros((0, cfg.dim), dt)
    c0, c1 = start // CHUNK, (start + count - 1) // CHUNK
    means = None if cfg.metric in CSR else _means(cfg)
    parts = []
    for c in range(c0, c1 + 1):
        r = _rng(cfg.data_seed, 2, c)
        parts.append(_csr_points(cfg, r, CHUNK) if cfg.metric in CSR else _mixture(cfg, means, r, CHUNK))
    lo = start - c0 * CHUNK
    if cfg.metric in CSR:
        allp = [s for p in parts for s in p]
        return allp[lo:lo + count]
    return np.concatenate(parts)[lo:lo + count]


def query_points(cfg: Config, count: int, seed_offset: int = 0):
    r = _rng(cfg.data_seed, 3, seed_offset)
    if cfg.metric in CSR:
        return _csr_points(cfg, r, count)
    return _mixture(cfg, _means(cfg), r, count)


def line_points(values, dtype=np.uint8):
    """1-D hand-worked examples: one coordinate per point."""
    return np.asarray(values, dtype=dtype).reshape(-1, 1)
