"""Thin ctypes binding of the C ABI in include/knng.h (argument marshalling only).

Every step of every call runs in the library's CUDA kernels (libknng.so, sm_100a).
There is no CPU path: if the shared library is missing or no CUDA device is present,
the calls raise.  Names follow the C ABI.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KNNG_LIB") or os.path.join(_HERE, "libknng.so")

KNNG_L2SQ_U8, KNNG_L2SQ_F32, KNNG_JACCARD_U32SET, KNNG_JARO_WINKLER, KNNG_COSINE_2GRAM = 0, 1, 2, 3, 4
ERRORS = {
    -1: "INVALID_ARG", -2: "INSUFFICIENT", -3: "EMPTY", -4: "CAPACITY_INFEAS", -5: "OOM",
    -6: "CUDA", -7: "NCCL", -8: "CAPACITY_EXCEEDED",
}


class KnngError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s (%d): %s" % (ERRORS.get(code, "?"), code, msg))
        self.code = code


class knng_points(C.Structure):
    _fields_ = [("metric", C.c_int32), ("dim", C.c_int32), ("n", C.c_int64), ("data", C.c_void_p),
                ("offsets", C.c_void_p), ("data_on_device", C.c_int32)]


class knng_params(C.Structure):
    _fields_ = [("speedup", C.c_double), ("expansion_num", C.c_uint32), ("expansion_den", C.c_uint32),
                ("depth", C.c_int32), ("seed", C.c_uint64), ("start_override", C.c_void_p),
                ("start_override_len", C.c_int32), ("full_scan", C.c_int32), ("route", C.c_int32)]


class knng_stats(C.Structure):
    _fields_ = [("search_evals", C.c_int64), ("search_starts", C.c_int64), ("search_skipped", C.c_int64),
                ("search_expansions", C.c_int64), ("ball_nodes", C.c_int64), ("proposals", C.c_int64),
                ("allpair_pairs", C.c_int64), ("kernel_launches", C.c_int64), ("ms_search", C.c_float),
                ("ms_allpairs", C.c_float), ("ms_update", C.c_float), ("ms_merge", C.c_float),
                ("ms_total", C.c_float)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class knng_runtime(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_unique_id", C.c_void_p), ("cuda_stream", C.c_void_p), ("capacity", C.c_int64)]


EXPORTS = ["graph_init", "graph_insert_batch", "graph_search", "partition_kmedoids", "graph_get_rows",
           "graph_get_partition", "graph_size", "graph_degree", "graph_free", "graph_last_error",
           "graph_ball_bound", "graph_insert_stage_search", "graph_insert_stage_update", "graph_insert_stage_commit",
           "graph_nccl_unique_id", "graph_world", "graph_recompute_medoids", "graph_insert_sequential"]

_lib = None


def load_library(path=LIB_PATH):
    """Load libknng.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError("libknng.so not built (%s): run __graft_entry__.build()" % path)
    L = C.CDLL(path)
    P = C.c_void_p
    L.graph_init.argtypes = [C.POINTER(knng_points), C.c_int32, C.POINTER(knng_runtime), C.POINTER(C.c_void_p)]
    L.graph_insert_batch.argtypes = [P, C.POINTER(knng_points), C.POINTER(knng_params), C.POINTER(C.c_int64),
                                     C.POINTER(knng_stats)]
    L.graph_insert_sequential.argtypes = [P, C.POINTER(knng_points), C.POINTER(knng_params), C.POINTER(C.c_int64),
                                          C.POINTER(knng_stats)]
    L.graph_search.argtypes = [P, C.POINTER(knng_points), C.c_int32, C.POINTER(knng_params), P, P, C.c_int32,
                               C.POINTER(knng_stats)]
    L.partition_kmedoids.argtypes = [P, C.c_int32, C.c_double, C.c_int32, C.c_uint64, P, P, P, P]
    L.graph_get_rows.argtypes = [P, C.c_int64, C.c_int64, P, P]
    L.graph_get_partition.argtypes = [P, P, P, C.POINTER(C.c_int32)]
    L.graph_size.argtypes = [P]
    L.graph_size.restype = C.c_int64
    L.graph_degree.argtypes = [P]
    L.graph_degree.restype = C.c_int32
    L.graph_free.argtypes = [P]
    L.graph_free.restype = None
    L.graph_last_error.restype = C.c_char_p
    L.graph_ball_bound.argtypes = [P, C.c_int32]
    L.graph_ball_bound.restype = C.c_int64
    L.graph_insert_stage_search.argtypes = [P, C.POINTER(knng_points), C.POINTER(knng_params), C.c_int32,
                                            C.c_int32, C.c_int64, C.c_int64, P, P, C.POINTER(knng_stats)]
    L.graph_insert_stage_update.argtypes = [P, C.POINTER(knng_params), C.c_int32, P, P, C.c_int64, C.c_int64, P, P,
                                            P, P, C.POINTER(knng_stats)]
    L.graph_insert_stage_commit.argtypes = [P, C.POINTER(knng_params), C.c_int64, P, P, P, P, C.POINTER(knng_stats)]
    L.graph_nccl_unique_id.argtypes = [P]
    L.graph_nccl_unique_id.restype = C.c_int
    L.graph_recompute_medoids.argtypes = [P, C.c_uint64, C.c_int64, P, C.POINTER(C.c_int64)]
    L.graph_recompute_medoids.restype = C.c_int
    L.graph_world.argtypes = [P]
    L.graph_world.restype = C.c_int32
    for f in ("graph_insert_stage_search", "graph_insert_stage_update", "graph_insert_stage_commit"):
        getattr(L, f).restype = C.c_int
    for f in ("graph_init", "graph_insert_batch", "graph_insert_sequential", "graph_search", "partition_kmedoids",
              "graph_get_rows", "graph_get_partition"):
        getattr(L, f).restype = C.c_int
    _lib = L
    return L


def _check(rc):
    if rc < 0:
        raise KnngError(rc, load_library().graph_last_error().decode())
    return rc


def _metric_of(arr):
    dt = np.dtype(str(arr.dtype).replace("torch.", ""))
    if dt == np.uint8:
        return KNNG_L2SQ_U8
    if dt == np.float32:
        return KNNG_L2SQ_F32
    raise TypeError("points must be uint8 or float32, got %s" % arr.dtype)


class TokenSets:
    """Jaccard sets in CSR form: offsets uint64[n+1], tokens uint32 (each set sorted, unique).
    Both host numpy arrays, or both CUDA torch tensors (int64 / int32 views are accepted)."""
    metric = KNNG_JACCARD_U32SET

    def __init__(self, offsets, tokens):
        self.offsets = offsets
        self.tokens = tokens

    @classmethod
    def from_list(cls, sets, **kw):
        off = np.zeros(len(sets) + 1, np.uint64)
        off[1:] = np.cumsum([len(x) for x in sets])
        tok = (np.concatenate([np.asarray(x, np.uint32) for x in sets]) if len(sets) else np.zeros(0, np.uint32))
        return cls(off, np.ascontiguousarray(tok, np.uint32), **kw)


class Strings(TokenSets):
    """Strings for KNNG_JARO_WINKLER / KNNG_COSINE_2GRAM in the same CSR form: one uint32 character per
    element, in string order (<= 127 per string).  from_list accepts python str or arrays of code units."""

    def __init__(self, offsets, chars, metric):
        super().__init__(offsets, chars)
        if metric not in (KNNG_JARO_WINKLER, KNNG_COSINE_2GRAM):
            raise ValueError("Strings: metric must be KNNG_JARO_WINKLER or KNNG_COSINE_2GRAM")
        self.metric = metric

    @classmethod
    def from_list(cls, strs, metric):
        arrs = [np.frombuffer(x.encode("utf-32-le"), np.uint32) if isinstance(x, str) else np.asarray(x, np.uint32)
                for x in strs]
        return super().from_list(arrs, metric=metric)

    def __len__(self):
        return len(self.offsets) - 1


def make_points(points, metric=None):
    """Marshal host numpy [n, dim] / CUDA torch [n, dim] vectors, Jaccard sets (a list of sorted uint32
    arrays or a TokenSets) or strings (a Strings, or a list with metric = a string metric) into
    knng_points.  Returns (struct, keepalive)."""
    if isinstance(points, list):
        points = (Strings.from_list(points, metric) if metric in (KNNG_JARO_WINKLER, KNNG_COSINE_2GRAM)
                  else TokenSets.from_list(points))
    if isinstance(points, TokenSets):
        o, t = points.offsets, points.tokens
        if hasattr(o, "is_cuda") and o.is_cuda:
            o, t = o.contiguous(), t.contiguous()
            p = knng_points(points.metric, 0, len(o) - 1, C.c_void_p(t.data_ptr() if t.numel() else 0),
                            C.c_void_p(o.data_ptr()), 1)
            return p, (o, t)
        o = np.ascontiguousarray(o, np.uint64)
        t = np.ascontiguousarray(t, np.uint32)
        if len(t) == 0:
            t = np.zeros(1, np.uint32)
        p = knng_points(points.metric, 0, len(o) - 1, t.ctypes.data_as(C.c_void_p),
                        o.ctypes.data_as(C.c_void_p), 0)
        return p, (o, t)
    if hasattr(points, "is_cuda") and points.is_cuda:
        t = points.contiguous()
        n, d = t.shape
        p = knng_points(_metric_of(t), d, n, C.c_void_p(t.data_ptr()), None, 1)
        return p, t
    a = np.ascontiguousarray(points)
    if a.ndim != 2:
        raise ValueError("points must be [n, dim]")
    n, d = a.shape
    p = knng_points(_metric_of(a), d, n, a.ctypes.data_as(C.c_void_p), None, 0)
    return p, a


def make_params(speedup, e_num, e_den, depth, seed, starts=None, full_scan=0, route=0):
    keep = None
    sp, sl = None, 0
    if starts is not None:
        keep = np.ascontiguousarray(starts, np.int32)
        sp, sl = keep.ctypes.data_as(C.c_void_p), len(keep)
    return knng_params(float(speedup), int(e_num), int(e_den), int(depth), int(seed), sp, sl, int(full_scan),
                       int(route)), keep


def nccl_unique_id():
    """A new 128-byte NCCL unique id (bytes) for KnngGraph(..., rank, world, nccl_id)."""
    buf = C.create_string_buffer(128)
    _check(load_library().graph_nccl_unique_id(buf))
    return buf.raw


class KnngGraph:
    """One graph handle (graph_init ... graph_free).  With world > 1 (or an nccl_id), the handle owns an
    NCCL communicator and insert_batch is the distributed insert (every rank passes the same batch)."""

    def __init__(self, points, k, device=0, capacity=0, stream=None, rank=0, world=1, nccl_id=None, metric=None):
        L = load_library()
        p, keep = make_points(points, metric)
        self._id = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), 128)
        rt = knng_runtime(int(device), int(rank), int(world),
                          None if self._id is None else C.cast(self._id, C.c_void_p),
                          C.c_void_p(stream) if stream else None, int(capacity))
        h = C.c_void_p()
        _check(L.graph_init(C.byref(p), int(k), C.byref(rt), C.byref(h)))
        del keep
        self._h = h
        self.k = int(k)
        self.metric = p.metric
        self.dim = p.dim

    def close(self):
        if getattr(self, "_h", None):
            load_library().graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def world(self):
        return int(load_library().graph_world(self._h))

    @property
    def n(self):
        return int(load_library().graph_size(self._h))

    def insert_batch(self, points, speedup, e_num, e_den, depth, seed, route=0):
        p, keep = make_points(points, self.metric)
        prm, _ = make_params(speedup, e_num, e_den, depth, seed, route=route)
        first = C.c_int64()
        st = knng_stats()
        _check(load_library().graph_insert_batch(self._h, C.byref(p), C.byref(prm), C.byref(first), C.byref(st)))
        return int(first.value), st.as_dict()

    def insert_sequential(self, points, speedup, e_num, e_den, depth, seed):
        """graph_insert_sequential: the points one after another, each a batch of one (the paper's
        sequential algorithm); one launch on an unpartitioned single-GPU graph."""
        p, keep = make_points(points, self.metric)
        prm, _ = make_params(speedup, e_num, e_den, depth, seed)
        first = C.c_int64()
        st = knng_stats()
        _check(load_library().graph_insert_sequential(self._h, C.byref(p), C.byref(prm), C.byref(first),
                                                      C.byref(st)))
        return int(first.value), st.as_dict()

    def search(self, queries, kr, speedup, e_num, e_den, seed, starts=None, out=None, full_scan=0, route=0):
        """graph_search: iGNNS; full_scan=1 with e_den=0 is the GNNS baseline; route=1 searches only
        the nearest medoid's partition (reading Q18's variant)."""
        p, keep = make_points(queries, self.metric)
        prm, keep2 = make_params(speedup, e_num, e_den, 1, seed, starts, full_scan, route)
        st = knng_stats()
        if out is not None:        # device outputs (torch int32 tensors)
            oi, ok = out
            _check(load_library().graph_search(self._h, C.byref(p), int(kr), C.byref(prm),
                                               C.c_void_p(oi.data_ptr()), C.c_void_p(ok.data_ptr()), 1,
                                               C.byref(st)))
            return oi, ok, st.as_dict()
        ids = np.zeros((p.n, kr), np.int32)
        keys = np.zeros((p.n, kr), np.uint32)
        _check(load_library().graph_search(self._h, C.byref(p), int(kr), C.byref(prm),
                                           ids.ctypes.data_as(C.c_void_p), keys.ctypes.data_as(C.c_void_p), 0,
                                           C.byref(st)))
        return ids, keys, st.as_dict()

    # ---- staged insert (multi-GPU building blocks; torch CUDA tensors) ----
    def ball_bound(self, depth):
        return int(load_library().graph_ball_bound(self._h, int(depth)))

    def stage_search(self, points, speedup, e_num, e_den, depth, seed, part_lo, part_hi, cand_ids, cand_keys,
                     q_lo=-1, q_hi=-1):
        p, keep = make_points(points, self.metric)
        prm, _ = make_params(speedup, e_num, e_den, depth, seed)
        st = knng_stats()
        _check(load_library().graph_insert_stage_search(self._h, C.byref(p), C.byref(prm), int(part_lo), int(part_hi),
                                                        int(q_lo), int(q_hi), C.c_void_p(cand_ids.data_ptr()),
                                                        C.c_void_p(cand_keys.data_ptr()), C.byref(st)))
        return st.as_dict()

    def stage_update(self, speedup, e_num, e_den, depth, seed, world, cand_ids_all, cand_keys_all, q_lo, q_hi, props,
                     prop_cnt, new_ids=None, new_keys=None):
        prm, _ = make_params(speedup, e_num, e_den, depth, seed)
        st = knng_stats()
        ptr = lambda t: None if t is None else C.c_void_p(t.data_ptr())
        _check(load_library().graph_insert_stage_update(self._h, C.byref(prm), int(world), ptr(cand_ids_all),
                                                        ptr(cand_keys_all), int(q_lo), int(q_hi), ptr(props),
                                                        ptr(prop_cnt), ptr(new_ids), ptr(new_keys), C.byref(st)))
        return st.as_dict()

    def stage_commit(self, speedup, e_num, e_den, depth, seed, nq_slots, props_all, prop_cnt_all, new_ids_all=None,
                     new_keys_all=None):
        prm, _ = make_params(speedup, e_num, e_den, depth, seed)
        st = knng_stats()
        ptr = lambda t: None if t is None else C.c_void_p(t.data_ptr())
        _check(load_library().graph_insert_stage_commit(self._h, C.byref(prm), int(nq_slots), ptr(props_all),
                                                        ptr(prop_cnt_all), ptr(new_ids_all), ptr(new_keys_all),
                                                        C.byref(st)))
        return st.as_dict()

    def partition_kmedoids(self, P, imbalance, max_iter, seed, init_medoids=None):
        n = self.n
        part = np.zeros(n, np.uint8)
        med = np.zeros(P, np.int32)
        cost = np.full(max_iter + 1, -1, np.int64)
        im = None if init_medoids is None else np.ascontiguousarray(init_medoids, np.int32)
        rc = _check(load_library().partition_kmedoids(
            self._h, int(P), float(imbalance), int(max_iter), int(seed), part.ctypes.data_as(C.c_void_p),
            med.ctypes.data_as(C.c_void_p), cost.ctypes.data_as(C.c_void_p),
            None if im is None else im.ctypes.data_as(C.c_void_p)))
        return part, med, cost[:rc]

    def rows(self, first=0, count=None):
        count = self.n - first if count is None else count
        ids = np.zeros((count, self.k), np.int32)
        keys = np.zeros((count, self.k), np.uint32)
        _check(load_library().graph_get_rows(self._h, int(first), int(count), ids.ctypes.data_as(C.c_void_p),
                                             keys.ctypes.data_as(C.c_void_p)))
        return ids, keys

    def recompute_medoids(self, seed, epoch):
        """graph_recompute_medoids (Alg. 5's last step): returns (medoids, total hop-sum cost)."""
        L = load_library()
        med = np.zeros(256, np.int32)
        cost = C.c_int64()
        _check(L.graph_recompute_medoids(self._h, int(seed), int(epoch), med.ctypes.data_as(C.c_void_p),
                                         C.byref(cost)))
        _, m = self.partition()
        return m, int(cost.value)

    def partition(self):
        P = C.c_int32()
        _check(load_library().graph_get_partition(self._h, None, None, C.byref(P)))
        if P.value == 0:
            return None, None
        part = np.zeros(self.n, np.uint8)
        med = np.zeros(P.value, np.int32)
        _check(load_library().graph_get_partition(self._h, part.ctypes.data_as(C.c_void_p),
                                                  med.ctypes.data_as(C.c_void_p), C.byref(P)))
        return part, med
