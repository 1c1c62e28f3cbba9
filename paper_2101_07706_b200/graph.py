"""Host-side graph types mirroring the reference's ``skewgcn.graph`` API surface.

``WeightedGraph`` keeps the reference's fields (graph.py:20-79) so a user's graph
object can be handed over unchanged; the device copy (int32 columns, fp64 weights,
owner map) is built lazily by :mod:`paper_2101_07706_b200._device` on first use.
The hot queries (``neighbor_union``, ``column_norms``, ``adjacency_block``) run on the
GPU through a saturated one-layer plan; there is no host implementation of them.
"""

from __future__ import annotations

import tempfile
from dataclasses import dataclass, replace
from pathlib import Path

import numpy as np
import scipy.sparse as sp


@dataclass
class WeightedGraph:
    """Undirected graph in canonical CSR form (rows sorted by neighbour id)."""

    n_nodes: int
    offsets: np.ndarray
    neighbors: np.ndarray
    weights: np.ndarray
    normalized: bool = False
    features: np.ndarray | None = None
    labels: np.ndarray | None = None
    train_mask: np.ndarray | None = None
    val_mask: np.ndarray | None = None
    test_mask: np.ndarray | None = None

    def __post_init__(self) -> None:
        # validation identical to graph.py:39-54
        self.offsets = np.asarray(self.offsets, dtype=np.int64)
        self.neighbors = np.asarray(self.neighbors, dtype=np.int64)
        self.weights = np.asarray(self.weights, dtype=np.float64)
        if self.offsets.shape != (self.n_nodes + 1,):
            raise ValueError("offsets must have length n_nodes + 1")
        if self.offsets[0] != 0 or self.offsets[-1] != len(self.neighbors):
            raise ValueError("offsets must start at 0 and end at len(neighbors)")
        if np.any(np.diff(self.offsets) < 0):
            raise ValueError("offsets must be nondecreasing")
        if len(self.neighbors) != len(self.weights):
            raise ValueError("neighbors and weights must be aligned")
        if len(self.neighbors) and (self.neighbors.min() < 0 or self.neighbors.max() >= self.n_nodes):
            raise ValueError("neighbor id out of range")

    @property
    def n_edges_stored(self) -> int:
        return len(self.neighbors)

    @property
    def feature_dim(self) -> int:
        if self.features is None:
            raise ValueError("graph carries no features")
        return self.features.shape[1]

    def row(self, i: int):
        lo, hi = self.offsets[i], self.offsets[i + 1]
        return self.neighbors[lo:hi], self.weights[lo:hi]

    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets)

    def to_sparse(self) -> sp.csr_matrix:
        return sp.csr_matrix((self.weights, self.neighbors, self.offsets),
                             shape=(self.n_nodes, self.n_nodes))


def node_set(ids) -> np.ndarray:
    """Sorted, duplicate-free int64 node ids (graph.py:82-87)."""
    arr = np.unique(np.asarray(ids, dtype=np.int64))
    if len(arr) and arr[0] < 0:
        raise ValueError("negative node id")
    return arr


def check_node_set(s, n_nodes: int) -> np.ndarray:
    """graph.py:90-98."""
    s = np.asarray(s, dtype=np.int64)
    if len(s) == 0:
        return s
    if np.any(np.diff(s) <= 0):
        raise ValueError("node set must be strictly increasing")
    if s[0] < 0 or s[-1] >= n_nodes:
        raise ValueError("node id out of range for this graph")
    return s


def _canonical_csr(src: np.ndarray, dst: np.ndarray, n_nodes: int):
    """Canonical CSR (sorted rows, deduplicated) from directed pairs (graph.py:101-112)."""
    if len(src) == 0:
        return np.zeros(n_nodes + 1, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros(0)
    key = np.sort(src.astype(np.int64) * n_nodes + dst.astype(np.int64))
    key = key[np.concatenate([[True], key[1:] != key[:-1]])]
    rows, cols = key // n_nodes, key % n_nodes
    offsets = np.zeros(n_nodes + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_nodes), out=offsets[1:])
    return offsets, cols, np.ones(len(key))


def graph_from_edges(edges, n_hint: int | None = None, normalize: bool = True) -> WeightedGraph:
    """Undirected edge list -> graph (each edge in both rows, duplicates collapsed)."""
    e = edges if isinstance(edges, np.ndarray) else np.asarray(list(edges), dtype=np.int64)
    e = np.asarray(e, dtype=np.int64).reshape(-1, 2)
    n = int(e.max()) + 1 if len(e) else 0
    if n_hint is not None:
        n = max(n, n_hint)
    if len(e) and e.min() < 0:
        raise ValueError("negative node id")
    offs, cols, w = _canonical_csr(np.concatenate([e[:, 0], e[:, 1]]),
                                   np.concatenate([e[:, 1], e[:, 0]]), n)
    g = WeightedGraph(n_nodes=n, offsets=offs, neighbors=cols, weights=w)
    return normalize_weights(g) if normalize else g


def load_edge_list(path, n_hint: int | None = None) -> WeightedGraph:
    """Edge-list text loader with the reference's rules (graph.py:115-149); vectorised,
    see datasets.load_edge_list."""
    from .datasets import load_edge_list as _load
    return _load(path, n_hint=n_hint)


def normalize_weights(g: WeightedGraph) -> WeightedGraph:
    """Self-loops and w_ij = 1/sqrt(d_i d_j) (graph.py:166-183); a one-off graph build."""
    if g.normalized:
        raise ValueError("graph is already normalized")
    n = g.n_nodes
    rows = np.repeat(np.arange(n, dtype=np.int64), g.degrees())
    loops = np.arange(n, dtype=np.int64)
    offs, cols, _ = _canonical_csr(np.concatenate([rows, loops]),
                                   np.concatenate([g.neighbors, loops]), n)
    deg = np.diff(offs).astype(np.float64)
    row_ids = np.repeat(np.arange(n, dtype=np.int64), np.diff(offs))
    w = 1.0 / np.sqrt(deg[row_ids] * deg[cols])
    return replace(g, offsets=offs, neighbors=cols, weights=w, normalized=True)


def undirected_edges(g: WeightedGraph) -> np.ndarray:
    rows = np.repeat(np.arange(g.n_nodes, dtype=np.int64), g.degrees())
    mask = rows <= g.neighbors
    return np.stack([rows[mask], g.neighbors[mask]], axis=1)


def from_shaped(sg) -> WeightedGraph:
    """Wrap a :class:`paper_2101_07706_b200.synth.ShapedGraph` without copying CSR data."""
    g = WeightedGraph.__new__(WeightedGraph)
    g.n_nodes = sg.n_nodes
    g.offsets = sg.offsets
    g.neighbors = sg.neighbors
    g.weights = sg.weights
    g.normalized = True
    g.features = sg.features
    g.labels = sg.labels
    g.train_mask = sg.train_mask
    g.val_mask = sg.val_mask
    g.test_mask = sg.test_mask
    return g


# ---- device-backed queries (a saturated one-layer plan; see _device.one_layer)

def neighbor_union(g: WeightedGraph, s) -> np.ndarray:
    """N(s) = union of adjacency rows of s, sorted (graph.py:186-195), on the GPU."""
    from ._device import one_layer, query_chunks
    s = check_node_set(s, g.n_nodes)
    if len(s) == 0:
        return np.zeros(0, dtype=np.int64)
    parts = [one_layer(g, c)["cand"].astype(np.int64) for c in query_chunks(g, s)]
    return parts[0] if len(parts) == 1 else np.unique(np.concatenate(parts))


_PUSH_MAX_ROWS = 16384  # row sets above this use the pull formulation


def column_norms(g: WeightedGraph, s_l, candidates) -> np.ndarray:
    """sum_{i in s_l} w_ij^2 per candidate, np.add.at order (graph.py:198-220), on the GPU."""
    from ._device import one_layer
    s_l = check_node_set(s_l, g.n_nodes)
    candidates = check_node_set(candidates, g.n_nodes)
    if len(s_l) == 0:
        if len(candidates):
            raise ValueError("candidates must be empty when s_l is empty")
        return np.zeros(0)
    from ._device import query_chunks
    if len(s_l) > _PUSH_MAX_ROWS or len(query_chunks(g, s_l)) > 1:
        # pull formulation: no per-call plan, any row count (a push plan holds < 2^16 pairs'
        # row ranks, and splitting the rows would reorder the np.add.at fold)
        from ._device import device_graph
        from ._native import check, lib, ptr
        import ctypes as C
        dg = device_graph(g)
        cand64 = np.ascontiguousarray(candidates, dtype=np.int64)
        rows64 = np.ascontiguousarray(s_l, dtype=np.int64)
        out = np.zeros(len(cand64), dtype=np.float64)
        check(lib.skg_column_norms_pull(dg.ctx, ptr(rows64, C.c_int64), len(rows64),
                                        ptr(cand64, C.c_int64), len(cand64), ptr(out, C.c_double)))
        return out
    lay = one_layer(g, s_l)
    cand, norm = lay["cand"].astype(np.int64), lay["norm"]
    pos = np.searchsorted(cand, candidates)
    pos_c = np.minimum(pos, len(cand) - 1)
    ok = cand[pos_c] == candidates
    out = np.where(ok, norm[pos_c], 0.0)
    if np.any(out <= 0.0):
        missing = candidates[out <= 0.0]
        raise ValueError(f"candidates not adjacent to s_l: {missing[:10].tolist()}")
    return out


def adjacency_block(g: WeightedGraph, rows, cols) -> sp.csr_matrix:
    """w[i, j] for i in rows, j in cols (graph.py:223-242); block built on the GPU."""
    from ._device import query_chunks
    rows = check_node_set(rows, g.n_nodes)
    cols = check_node_set(cols, g.n_nodes)
    if len(rows) == 0 or len(cols) == 0:
        return sp.csr_matrix((len(rows), len(cols)))
    parts = [_block_rows(g, c, cols) for c in query_chunks(g, rows)]
    return parts[0] if len(parts) == 1 else sp.vstack(parts, format="csr")


def _block_rows(g: WeightedGraph, rows, cols) -> sp.csr_matrix:
    from ._device import one_layer
    lay = one_layer(g, rows)
    full = lay["block"]                       # rows x N(rows), values w (p = 1)
    cand = lay["cand"].astype(np.int64)
    pos = np.searchsorted(cols, cand)
    pos_c = np.minimum(pos, len(cols) - 1)
    keep_col = cols[pos_c] == cand            # N(rows) columns that are requested
    remap = np.where(keep_col, pos_c, -1)
    new_idx = remap[full.indices]
    keep = new_idx >= 0
    row_of = np.repeat(np.arange(len(rows)), np.diff(full.indptr))
    counts = np.bincount(row_of[keep], minlength=len(rows))
    indptr = np.concatenate([[0], np.cumsum(counts)])
    return sp.csr_matrix((full.data[keep], new_idx[keep], indptr), shape=(len(rows), len(cols)))
