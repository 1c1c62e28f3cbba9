"""Device residency for the drop-in API: graph stores, plan-set pools, GCN workspaces.

A ``WeightedGraph`` gets one ``DeviceGraph`` (libskg context) the first time a hot
function sees it; partitions only re-upload the owner map.  Plan sets are pooled by
shape and leased to the ``SamplePlan`` objects that own their device data, so plans
stay valid while referenced (like the reference's immutable SamplePlan objects).
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref

import numpy as np

from ._native import DT, KIND_LADIES, KIND_SAINT, check, lib, ptr, require_device
from .features import BitFeatures, auto_pack

_COMPUTE = {"dtype": "float64"}


def set_compute_dtype(dtype: str) -> None:
    """'float64' (reference precision, default for the drop-in API) or 'float32'."""
    if dtype not in DT:
        raise ValueError(f"unknown dtype {dtype!r}")
    _COMPUTE["dtype"] = dtype


def compute_dtype() -> str:
    return _COMPUTE["dtype"]


def current_stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def pack_multihot(y: np.ndarray) -> np.ndarray:
    """n x C 0/1 matrix -> n x ceil(C/64) uint64 words (bit k%64 of word k/64 = class k)."""
    y = np.asarray(y) != 0
    n, c = y.shape
    nw = (c + 63) // 64
    pad = np.zeros((n, nw * 64), dtype=bool)
    pad[:, :c] = y
    weight = np.left_shift(np.uint64(1), np.arange(64, dtype=np.uint64))
    return np.ascontiguousarray((pad.reshape(n, nw, 64).astype(np.uint64) * weight).sum(axis=2,
                                                                                      dtype=np.uint64))


class PlanSet:
    """One skg_plans arena (n_slots plans) and its GCN workspaces."""

    def __init__(self, dg: "DeviceGraph", kind: int, n_slots: int, n_layers: int, budget: int,
                 max_batch: int):
        self.dg = dg
        self.kind, self.n_slots, self.n_layers = kind, n_slots, n_layers
        self.budget, self.max_batch = budget, max_batch
        h = C.c_void_p()
        check(lib.skg_plans_create(dg.ctx, kind, n_slots, n_layers, budget, max_batch, C.byref(h)))
        self.h = h
        self._gcn = {}
        self.train_key = None

    def key(self):
        return (self.kind, self.n_slots, self.n_layers, self.budget, self.max_batch)

    def gcn(self, dims, dtype: str):
        k = (tuple(int(d) for d in dims), dtype)
        if k not in self._gcn:
            g = C.c_void_p()
            d = np.asarray(dims, dtype=np.int64)
            check(lib.skg_gcn_create(self.h, len(dims) - 1, ptr(d, C.c_int64), DT[dtype], C.byref(g)))
            self._gcn[k] = g
        return self._gcn[k]

    def stats(self, slot: int = 0):
        st = np.zeros((self.n_layers, 16), dtype=np.int64)
        info = np.zeros(4, dtype=np.int64)
        rc = lib.skg_plan_stats(self.h, slot, ptr(st, C.c_int64), ptr(info, C.c_int64))
        return st, info, rc

    def destroy(self):
        for g in self._gcn.values():
            lib.skg_gcn_destroy(g)
        self._gcn.clear()
        if self.h:
            lib.skg_plans_destroy(self.h)
            self.h = None


class DeviceGraph:
    def __init__(self, g, device: int = 0):
        require_device()
        import torch  # noqa: F401  (CUDA context shared with torch)
        self.n = int(g.n_nodes)
        offs = np.ascontiguousarray(g.offsets, dtype=np.int64)
        nb = np.asarray(g.neighbors)
        if nb.dtype != np.int32:
            if len(nb) and nb.max() >= 2 ** 31:
                raise ValueError("node ids must fit in int32")
            nb = nb.astype(np.int32)
        nb = np.ascontiguousarray(nb)
        w = np.ascontiguousarray(g.weights, dtype=np.float64)
        own = np.zeros(max(self.n, 1), dtype=np.int32)
        h = C.c_void_p()
        check(lib.skg_ctx_create(device, self.n, len(nb), ptr(offs, C.c_int64), ptr(nb, C.c_int32),
                                 ptr(w, C.c_double), 1, ptr(own, C.c_int32), C.byref(h)))
        self.ctx = h
        self.device = device
        self.owner_key = None
        self.owner_ref = None
        self.feat_key = None
        self.feat_ref = None
        self.xbits = False
        self.lab_key = None
        self.lab_ref = None
        self.pool: dict = {}
        self.lock = threading.Lock()

    def __del__(self):
        try:
            for sets in self.pool.values():
                for ps in sets:
                    ps.destroy()
            if self.ctx:
                lib.skg_ctx_destroy(self.ctx)
        except Exception:
            pass

    # -- inputs -----------------------------------------------------------
    def ensure_owner(self, partition) -> None:
        owner = partition.owner
        key = (id(owner), owner.ctypes.data, owner.shape, int(partition.n_workers))
        if key == self.owner_key:
            return
        o32 = np.ascontiguousarray(owner, dtype=np.int32)
        if len(o32) != self.n:
            raise ValueError("partition size does not match the graph")
        check(lib.skg_ctx_set_owner(self.ctx, int(partition.n_workers), ptr(o32, C.c_int32)))
        self.owner_key, self.owner_ref = key, owner
        for sets in self.pool.values():  # SAINT local candidate lists depend on ownership
            for ps in sets:
                ps.train_key = None

    def ensure_features(self, X, dtype: str) -> None:
        """Upload the feature matrix: dense rows, or bit-packed rows for 0/1 (multi-hot)
        features (a BitFeatures matrix, or a dense 0/1 one at least 256 wide)."""
        if isinstance(X, BitFeatures):
            key = ("bits", id(X), X.words.ctypes.data, X.shape, dtype)
        else:
            key = (id(X), X.__array_interface__["data"][0], X.shape, str(X.dtype), dtype)
        if key == self.feat_key:
            return
        if X.shape[0] != self.n:
            raise ValueError(f"feature rows ({X.shape[0]}) != n_nodes ({self.n})")
        if auto_pack(X):
            bf = X if isinstance(X, BitFeatures) else BitFeatures.from_dense(X)
            check(lib.skg_ctx_set_features_bits(self.ctx, DT[dtype], bf.dim, bf.shape[0],
                                                bf.words.ctypes.data_as(C.c_void_p), bf.words.shape[1]))
            self.xbits = True
        else:
            host = np.ascontiguousarray(X, dtype=np.float32 if dtype == "float32" else np.float64)
            check(lib.skg_ctx_set_features(self.ctx, DT[dtype], host.shape[1], host.shape[0],
                                           host.ctypes.data_as(C.c_void_p)))
            self.xbits = False
        self.feat_key, self.feat_ref = key, X
        for sets in self.pool.values():
            for ps in sets:
                for g in ps._gcn.values():
                    lib.skg_gcn_destroy(g)
                ps._gcn.clear()

    def set_feature_shards(self, shard_ptrs, node_rank: np.ndarray, node_row: np.ndarray) -> None:
        """Route layer-0 gathers through a table of shard base pointers (this rank's shard
        or NVLink-mapped peer shards): node -> (rank, row).  Shards use the same padded row
        stride and dtype as the features set with ensure_features."""
        p = np.ascontiguousarray(np.asarray(shard_ptrs, dtype=np.uint64))
        r = np.ascontiguousarray(node_rank, dtype=np.int32)
        w = np.ascontiguousarray(node_row, dtype=np.int32)
        if len(r) != self.n or len(w) != self.n:
            raise ValueError("node_rank/node_row must cover every node")
        check(lib.skg_ctx_set_feature_map(self.ctx, len(p), ptr(p, C.c_uint64), ptr(r, C.c_int32),
                                          ptr(w, C.c_int32)))

    def upload_shard(self, rows: np.ndarray, dtype: str) -> int:
        """Copy host feature rows into their own device allocation (IPC-exportable)."""
        if self.xbits:  # the store holds packed rows: upload the shard packed too
            bf = rows if isinstance(rows, BitFeatures) else BitFeatures.from_dense(rows)
            host = bf.words
        else:
            host = np.ascontiguousarray(rows, dtype=np.float32 if dtype == "float32" else np.float64)
        out = C.c_uint64()
        check(lib.skg_ctx_shard_upload(self.ctx, host.ctypes.data_as(C.c_void_p), host.shape[0],
                                       C.byref(out)))
        return int(out.value)

    def feature_ld(self) -> int:
        out = C.c_uint64()
        ld = C.c_int64()
        check(lib.skg_ctx_feature_ptr(self.ctx, C.byref(out), C.byref(ld)))
        return int(ld.value)

    def ensure_labels(self, labels: np.ndarray) -> None:
        """Class per node (1-D, -1 = unlabeled), or an n x C multi-hot matrix for the
        multi-label BCE loss (packed into 64-bit words per node)."""
        key = (id(labels), labels.__array_interface__["data"][0], labels.shape)
        if key == self.lab_key:
            return
        if labels.ndim == 2:
            words = pack_multihot(labels)
            check(lib.skg_ctx_set_multilabels(self.ctx, ptr(words, C.c_uint64), labels.shape[1]))
        else:
            l64 = np.ascontiguousarray(labels, dtype=np.int64)
            check(lib.skg_ctx_set_labels(self.ctx, ptr(l64, C.c_int64)))
        self.lab_key, self.lab_ref = key, labels

    # -- plan-set pool ----------------------------------------------------
    def acquire(self, kind, n_slots, n_layers, budget, max_batch) -> PlanSet:
        key = (kind, n_slots, n_layers, budget, max_batch)
        with self.lock:
            free = self.pool.setdefault(key, [])
            for ps in free:
                if not getattr(ps, "leased", False):
                    ps.leased = True
                    return ps
            ps = PlanSet(self, kind, n_slots, n_layers, budget, max_batch)
            ps.leased = True
            free.append(ps)
            if len(free) > 8:  # bound pooled memory
                for old in [p for p in free if not p.leased][: len(free) - 8]:
                    old.destroy()
                    free.remove(old)
            return ps

    def release(self, ps: PlanSet) -> None:
        ps.leased = False


def device_graph(g) -> DeviceGraph:
    dg = g.__dict__.get("_skg_dev")
    if dg is None or dg.n != g.n_nodes:
        dg = DeviceGraph(g)
        g.__dict__["_skg_dev"] = dg
    return dg


class Lease:
    """Keeps a PlanSet slot alive while a SamplePlan references it."""

    def __init__(self, dg: DeviceGraph, ps: PlanSet, slot: int = 0):
        self.dg, self.ps, self.slot = dg, ps, slot
        self._fin = weakref.finalize(self, dg.release, ps)


def read_layer(ps: PlanSet, slot: int, t: int, st_row: np.ndarray, want_dist: bool):
    n_upper, n_cand, n_nodes, nnz = (int(x) for x in st_row[:4])
    nodes = np.zeros(max(n_nodes, 1), dtype=np.int32)
    indptr = np.zeros(n_upper + 1, dtype=np.int32)
    indices = np.zeros(max(nnz, 1), dtype=np.int32)
    values = np.zeros(max(nnz, 1), dtype=np.float64)
    cand = np.zeros(max(n_cand, 1), dtype=np.int32) if want_dist else None
    norm = np.zeros(max(n_cand, 1), dtype=np.float64) if want_dist else None
    loc = np.zeros(max(n_cand, 1), dtype=np.uint8) if want_dist else None
    null = lambda a, t_: ptr(a, t_) if a is not None else None  # noqa: E731
    check(lib.skg_plan_layer(ps.h, slot, t, ptr(nodes, C.c_int32), ptr(indptr, C.c_int32),
                             ptr(indices, C.c_int32), ptr(values, C.c_double),
                             null(cand, C.c_int32), null(norm, C.c_double), null(loc, C.c_uint8)))
    out = {"nodes": nodes[:n_nodes].astype(np.int64), "indptr": indptr, "indices": indices[:nnz],
           "values": values[:nnz], "shape": (n_upper, n_nodes)}
    if want_dist:
        out.update(cand=cand[:n_cand], norm=norm[:n_cand], is_local=loc[:n_cand].astype(bool))
    return out


_RANK_LIMIT = 65535  # LADIES plans keep upper-row ranks / pair counters in 16 bits


def _pow2(x: int) -> int:
    return 1 << max(0, int(x) - 1).bit_length()


def query_chunks(g, s: np.ndarray):
    """Split a sorted row set into consecutive runs a saturated one-layer plan can hold
    (rows and the sum of their degrees both below the 16-bit rank limit)."""
    deg = np.diff(np.asarray(g.offsets))[s]
    if len(s) and int(deg.max()) >= _RANK_LIMIT:
        raise ValueError("a row's degree exceeds the device query limit (65534)")
    out, lo, acc = [], 0, 0
    for i, d in enumerate(deg.tolist()):
        if i > lo and (acc + d >= _RANK_LIMIT or i - lo >= _RANK_LIMIT - 1):
            out.append(s[lo:i])
            lo, acc = i, 0
        acc += d
    if len(s):
        out.append(s[lo:])
    return out


def one_layer(g, s: np.ndarray) -> dict:
    """Saturated single-layer plan over upper set s: N(s), column norms, block (p = 1).
    The budget is min(n, sum of deg(s)) >= |N(s)|, so the layer never draws; callers
    split row sets beyond the 16-bit rank limit with ``query_chunks``."""
    import scipy.sparse as sp
    dg = device_graph(g)
    bound = int(np.diff(np.asarray(g.offsets))[s].sum()) if len(s) else 1
    budget = max(1, min(int(g.n_nodes), bound))
    if max(budget, len(s)) >= _RANK_LIMIT:
        raise ValueError("row set too large for one device query; split it with query_chunks")
    # pooled arenas are keyed by shape: round to powers of two so repeated queries of
    # different sizes share a few arenas
    budget_k = min(_pow2(budget), _RANK_LIMIT - 1, max(int(g.n_nodes), 1))
    ps = dg.acquire(KIND_LADIES, 1, 1, budget_k, min(_pow2(max(len(s), 1)), _RANK_LIMIT - 1))
    try:
        off = np.array([0, len(s)], dtype=np.int64)
        ids = np.ascontiguousarray(s, dtype=np.int64)
        w = np.zeros(1, dtype=np.int32)
        rng = np.zeros(4, dtype=np.uint64)
        check(lib.skg_ladies_sample(ps.h, 1, ptr(w, C.c_int32), ptr(off, C.c_int64),
                                    ptr(ids, C.c_int64), 0, 0.0, 1.0, ptr(rng, C.c_uint64), None))
        st, info, rc = ps.stats(0)
        check(rc)
        lay = read_layer(ps, 0, 0, st[0], True)
        lay["block"] = sp.csr_matrix((lay["values"], lay["indices"], lay["indptr"]),
                                     shape=lay["shape"])
        return lay
    finally:
        dg.release(ps)
