"""CPU oracle for the skewed layer-wise sampling hot path (TEST INFRASTRUCTURE ONLY).

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The product path
(``paper_2101_07706_b200``) never imports anything under ``oracle/`` and
fails loudly when its CUDA library is missing.

It restates, in plain numpy/scipy, the algorithm of the reference package
``skewgcn`` (arXiv 2101.07706 simulator, mounted read-only at
``/root/reference/pkg/src/skewgcn``).  Every function cites the reference
``file:line`` it follows.  The arithmetic that decides bit-exactness is kept
operation-for-operation identical to the reference (numpy's sequential
``np.add.at`` fold, its pairwise ``sum``, the ``cumsum``/``searchsorted``
decomposition of ``Generator.choice``, multiply-by-reciprocal block values).

Parity pin: ``tests/test_oracle_golden.py`` checks this restatement against
golden vectors produced by the unmodified reference itself
(``tests/golden/make_golden.py``, run in the build container where the
reference is importable), so the oracle is *pinned*, not self-certified.

Pinned third-party behaviour (un-vendored in the reference,
``pkg/pyproject.toml:10-13`` gives only lower bounds): numpy 2.3.5,
scipy 1.18.1 — the versions in this image.
"""

from __future__ import annotations

import hashlib
import warnings
from dataclasses import dataclass, field, replace

import numpy as np
import scipy.sparse as sp

# ---------------------------------------------------------------------------
# Graph store (reference: graph.py)
# ---------------------------------------------------------------------------


@dataclass
class Graph:
    """Canonical CSR graph; mirrors ``WeightedGraph`` (graph.py:20-79)."""

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

    def __post_init__(self):
        self.offsets = np.asarray(self.offsets, dtype=np.int64)
        self.neighbors = np.asarray(self.neighbors, dtype=np.int64)
        self.weights = np.asarray(self.weights, dtype=np.float64)

    def degrees(self):
        return np.diff(self.offsets)

    @property
    def feature_dim(self):
        return self.features.shape[1]

    def to_sparse(self):
        # graph.py:74-79
        return sp.csr_matrix((self.weights, self.neighbors, self.offsets),
                             shape=(self.n_nodes, self.n_nodes))


def node_set(ids) -> np.ndarray:
    """graph.py:82-87 — sorted unique int64, negative ids rejected."""
    out = np.unique(np.asarray(ids, dtype=np.int64))
    if out.size and out[0] < 0:
        raise ValueError("negative node id")
    return out


def check_node_set(s, n_nodes: int) -> np.ndarray:
    """graph.py:90-98."""
    s = np.asarray(s, dtype=np.int64)
    if s.size == 0:
        return s
    if np.any(s[1:] <= s[:-1]):
        raise ValueError("node set must be strictly increasing")
    if s[0] < 0 or s[-1] >= n_nodes:
        raise ValueError("node id out of range for this graph")
    return s


def csr_from_pairs(src, dst, n_nodes: int):
    """graph.py:101-112 — dedup via a sorted key, counts via add.at."""
    if len(src) == 0:
        return (np.zeros(n_nodes + 1, dtype=np.int64), np.zeros(0, dtype=np.int64),
                np.zeros(0))
    key = np.unique(np.asarray(src, np.int64) * n_nodes + np.asarray(dst, np.int64))
    row, col = key // n_nodes, key % n_nodes
    offs = np.zeros(n_nodes + 1, dtype=np.int64)
    np.add.at(offs, row + 1, 1)
    np.cumsum(offs, out=offs)
    return offs, col, np.ones(len(key))


def graph_from_edge_array(edges, n_nodes: int) -> Graph:
    """Undirected edge pairs -> un-normalized canonical CSR (graph.py:144-149)."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    u, v = e[:, 0], e[:, 1]
    offs, col, w = csr_from_pairs(np.concatenate([u, v]), np.concatenate([v, u]), n_nodes)
    return Graph(n_nodes=n_nodes, offsets=offs, neighbors=col, weights=w)


def normalize_weights(g: Graph) -> Graph:
    """graph.py:166-183 — self-loops, w_ij = 1/sqrt(d_i*d_j), d counts the loop."""
    if g.normalized:
        raise ValueError("graph is already normalized")
    n = g.n_nodes
    rows = np.repeat(np.arange(n, dtype=np.int64), g.degrees())
    loop = np.arange(n, dtype=np.int64)
    offs, col, _ = csr_from_pairs(np.concatenate([rows, loop]),
                                  np.concatenate([g.neighbors, loop]), n)
    d = np.diff(offs).astype(np.float64)
    r = np.repeat(np.arange(n, dtype=np.int64), np.diff(offs))
    w = 1.0 / np.sqrt(d[r] * d[col])
    return replace(g, offsets=offs, neighbors=col, weights=w, normalized=True)


def _rows(g: Graph, s: np.ndarray):
    """Concatenated (columns, weights) of the CSR rows of s, in order of s."""
    if len(s) == 0:
        return np.zeros(0, np.int64), np.zeros(0), np.zeros(0, np.int64)
    lo, hi = g.offsets[s], g.offsets[s + 1]
    lens = hi - lo
    # vectorised equivalent of concatenating g.neighbors[lo:hi] per row
    base = np.repeat(lo - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
    idx = base + np.arange(lens.sum(), dtype=np.int64)
    return g.neighbors[idx], g.weights[idx], lens


def neighbor_union(g: Graph, s) -> np.ndarray:
    """graph.py:186-195 — N(s), sorted and deduplicated."""
    s = check_node_set(s, g.n_nodes)
    if len(s) == 0:
        return np.zeros(0, dtype=np.int64)
    cols, _, _ = _rows(g, s)
    return np.unique(cols)


def column_norms(g: Graph, s_l, candidates) -> np.ndarray:
    """graph.py:198-220 — sum_{i in s_l} w_ij^2 per candidate.

    The fold is ``np.add.at`` in contribution order (i ascending, then j
    ascending within a row), starting from 0.0: this order is what the CUDA
    kernel reproduces bit-for-bit.
    """
    s_l = check_node_set(s_l, g.n_nodes)
    candidates = check_node_set(candidates, g.n_nodes)
    if len(s_l) == 0:
        if len(candidates):
            raise ValueError("candidates must be empty when s_l is empty")
        return np.zeros(0)
    acc = np.zeros(len(candidates))
    cols, w, _ = _rows(g, s_l)
    pos = np.minimum(np.searchsorted(candidates, cols), len(candidates) - 1)
    hit = candidates[pos] == cols
    np.add.at(acc, pos[hit], w[hit] * w[hit])
    if np.any(acc <= 0.0):
        bad = candidates[acc <= 0.0]
        raise ValueError(f"candidates not adjacent to s_l: {bad[:10].tolist()}")
    return acc


def adjacency_block(g: Graph, rows, cols) -> sp.csr_matrix:
    """graph.py:223-242 — w[i, j] for i in rows, j in cols, canonical CSR."""
    rows = check_node_set(rows, g.n_nodes)
    cols = check_node_set(cols, g.n_nodes)
    if len(rows) == 0 or len(cols) == 0:
        return sp.csr_matrix((len(rows), len(cols)))
    nb, w, lens = _rows(g, rows)
    pos = np.minimum(np.searchsorted(cols, nb), len(cols) - 1)
    hit = cols[pos] == nb
    row_of = np.repeat(np.arange(len(rows)), lens)
    indptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.add.at(indptr, row_of[hit] + 1, 1)
    np.cumsum(indptr, out=indptr)
    return sp.csr_matrix((w[hit], pos[hit], indptr), shape=(len(rows), len(cols)))


# ---------------------------------------------------------------------------
# Partition and seeding (reference: partition.py, seeding.py)
# ---------------------------------------------------------------------------


def spawn_rng(master_seed: int, *labels) -> np.random.Generator:
    """seeding.py:17-27 — SHA-256 label words -> SeedSequence -> PCG64."""
    ent = [master_seed & 0xFFFFFFFFFFFFFFFF]
    for lab in labels:
        dig = hashlib.sha256(repr(lab).encode("utf-8")).digest()
        ent += [int.from_bytes(dig[o:o + 4], "little") for o in (0, 4, 8, 12)]
    return np.random.default_rng(np.random.SeedSequence(ent))


@dataclass
class Partition:
    """partition.py:16-40."""

    n_workers: int
    owner: np.ndarray

    def __post_init__(self):
        self.owner = np.asarray(self.owner, dtype=np.int64)

    def owned_by(self, w: int) -> np.ndarray:
        return np.flatnonzero(self.owner == w).astype(np.int64)


def partition_nodes(n: int, k: int, strategy: str = "contiguous", seed=None) -> Partition:
    """partition.py:43-74 (first n % k workers take the extra node)."""
    counts = np.full(k, n // k, dtype=np.int64)
    counts[: n % k] += 1
    chunked = np.repeat(np.arange(k, dtype=np.int64), counts)
    if strategy == "contiguous":
        owner = chunked
    elif strategy == "hash":
        owner = np.arange(n, dtype=np.int64) % k
    elif strategy == "random":
        perm = spawn_rng(seed, "partition").permutation(n)
        owner = np.empty(n, dtype=np.int64)
        owner[perm] = chunked
    else:
        raise ValueError(f"unknown strategy {strategy!r}")
    return Partition(k, owner)


def local_mask(nodes, part: Partition, worker: int) -> np.ndarray:
    """partition.py:111-115."""
    if not 0 <= worker < part.n_workers:
        raise ValueError("worker id out of range")
    return part.owner[np.asarray(nodes, dtype=np.int64)] == worker


# ---------------------------------------------------------------------------
# Sampling distributions (reference: sampling.py)
# ---------------------------------------------------------------------------


@dataclass
class SamplerConfig:
    """sampling.py:25-49."""

    budget: int
    skew_constant: float = 0.0
    mode: str = "full"
    min_scale: float = 1.0


@dataclass
class Dist:
    """ProbDist (sampling.py:52-75)."""

    candidates: np.ndarray
    q: np.ndarray
    is_local: np.ndarray
    s_used: float = 1.0


def skew_scale(D: float, n_cand: int, budget: int, n_remote: int, min_scale: float = 1.0):
    """sampling.py:126-138 — max(min_scale, D*(N-B)/R + 1/2), Python float ops."""
    if n_remote <= 0:
        raise ValueError("no remote candidates; use linear weights instead")
    raw = D * (n_cand - budget) / n_remote + 0.5
    return max(min_scale, raw)


def linear_dist(cands, norms, flags) -> Dist:
    """sampling.py:95-107 — q = norm / pairwise_sum(norm)."""
    norms = np.asarray(norms, dtype=np.float64)
    return Dist(cands, norms / norms.sum(), np.asarray(flags, bool), 1.0)


def skewed_dist(cands, norms, flags, s: float) -> Dist:
    """sampling.py:110-123 — local mass multiplied by s, then normalised."""
    norms = np.asarray(norms, dtype=np.float64)
    flags = np.asarray(flags, dtype=bool)
    scaled = np.where(flags, s * norms, norms)
    return Dist(cands, scaled / scaled.sum(), flags, float(s))


def inclusion_probability(q, budget: int):
    """sampling.py:166-179 — p = -expm1(B * log1p(-q))."""
    q = np.asarray(q, dtype=np.float64)
    with np.errstate(divide="ignore"):
        return -np.expm1(budget * np.log1p(-q))


def categorical_draws(q: np.ndarray, budget: int, rng: np.random.Generator) -> np.ndarray:
    """``rng.choice(len(q), budget, replace=True, p=q)`` (sampling.py:184) restated.

    numpy's Generator.choice with p and replacement is exactly: a strictly
    sequential ``cumsum``, division by its last element, ``budget`` uniforms
    ``(next_u64 >> 11) * 2**-53`` and ``searchsorted(..., side='right')``
    (verified bit-equal in this image).
    """
    cdf = q.cumsum()
    cdf /= cdf[-1]
    u = rng.random(budget)
    return cdf.searchsorted(u, side="right")


def sample_layer(cands, norms, flags, cfg: SamplerConfig, rng):
    """training.py:145-159 + draw_sample (sampling.py:182-191)."""
    if cfg.budget >= len(cands):
        return cands, np.ones(len(cands)), None
    if cfg.mode == "skewed" and np.any(~flags):
        s = skew_scale(cfg.skew_constant, len(cands), cfg.budget,
                       int(np.sum(~flags)), cfg.min_scale)
        dist = skewed_dist(cands, norms, flags, s)
    else:
        dist = linear_dist(cands, norms, flags)
    picks = np.unique(categorical_draws(dist.q, cfg.budget, rng))
    p_all = inclusion_probability(dist.q, cfg.budget)
    return cands[picks], p_all[picks], dist


# ---------------------------------------------------------------------------
# Plans (reference: training.py:81-254)
# ---------------------------------------------------------------------------


@dataclass
class Layer:
    nodes: np.ndarray
    block: sp.csr_matrix
    dist: Dist | None
    remote_sampled: int


@dataclass
class Plan:
    layers: list
    batch: np.ndarray
    starvation_events: int = 0

    @property
    def n_layers(self):
        return len(self.layers)

    @property
    def input_nodes(self):
        return self.layers[0].nodes

    def remote_per_layer(self):
        return np.array([L.remote_sampled for L in self.layers], dtype=np.int64)


def reweighted_block(g, upper, sampled, p):
    """training.py:137-142 — entries w_ij * (1/p_j) (multiply by reciprocal)."""
    blk = adjacency_block(g, upper, sampled)
    if len(sampled):
        recip = 1.0 / np.asarray(p, dtype=np.float64)
        blk = sp.csr_matrix((blk.data * recip[blk.indices], blk.indices, blk.indptr),
                            shape=blk.shape)
    return blk


def ladies_plan(g, part, worker, batch, cfg: SamplerConfig, n_layers, rng) -> Plan:
    """training.py:162-208 — top-down layer-wise sampling, then reversed."""
    batch = node_set(batch)
    if len(batch) == 0:
        raise ValueError("empty batch")
    upper, out, starved = batch, [], 0
    for _ in range(n_layers):
        cands = neighbor_union(g, upper)
        if cfg.mode == "local":
            cands = cands[local_mask(cands, part, worker)]
            if len(cands):
                hits = adjacency_block(g, upper, cands)
                starved += int(np.sum(np.diff(hits.indptr) == 0))
            else:
                starved += len(upper)
        if len(cands) == 0:
            out.append(Layer(cands, sp.csr_matrix((len(upper), 0)), None, 0))
            upper = cands
            continue
        norms = column_norms(g, upper, cands)
        flags = local_mask(cands, part, worker)
        picked, p, dist = sample_layer(cands, norms, flags, cfg, rng)
        remote = int(np.sum(~local_mask(picked, part, worker)))
        out.append(Layer(picked, reweighted_block(g, upper, picked, p), dist, remote))
        upper = picked
    out.reverse()
    return Plan(out, batch, starved)


def saint_plan(g, part, worker, train_nodes, subgraph_size, cfg: SamplerConfig,
               n_layers, rng, norms=None) -> Plan:
    """training.py:216-254 — one subgraph over training nodes, reused per layer."""
    train_nodes = node_set(train_nodes)
    if len(train_nodes) == 0:
        raise ValueError("empty training node set")
    if subgraph_size > len(train_nodes):
        warnings.warn("subgraph size exceeds training set; clamping")
        subgraph_size = len(train_nodes)
    if subgraph_size < 1:
        raise ValueError("subgraph size must be >= 1")
    cands = train_nodes
    flags = local_mask(cands, part, worker)
    if cfg.mode == "local":
        cands = cands[flags]
        if len(cands) == 0:
            raise ValueError("no local training nodes to sample a subgraph from")
        flags = np.ones(len(cands), dtype=bool)
        norms = None
        subgraph_size = min(subgraph_size, len(cands))
    if norms is None:
        norms = column_norms(g, train_nodes, cands)
    sub, p, dist = sample_layer(cands, norms, flags, replace(cfg, budget=subgraph_size), rng)
    blk = reweighted_block(g, sub, sub, p)
    remote = int(np.sum(~local_mask(sub, part, worker)))
    layers = [Layer(sub, blk, dist, remote if l == 0 else 0) for l in range(n_layers)]
    return Plan(layers, sub)


# ---------------------------------------------------------------------------
# GCN model, forward/backward (reference: training.py:40-74, 261-318)
# ---------------------------------------------------------------------------


def init_model(dims, seed):
    """training.py:65-74 — Glorot uniform from spawn_rng(seed, 'init', l)."""
    ws = []
    for l, (a, b) in enumerate(zip(dims, dims[1:])):
        bound = np.sqrt(6.0 / (a + b))
        ws.append(spawn_rng(seed, "init", l).uniform(-bound, bound, size=(a, b)))
    return ws


def forward(weights, plan: Plan, features):
    """training.py:261-269."""
    h = features[plan.input_nodes]
    for l, (L, w) in enumerate(zip(plan.layers, weights)):
        a = np.maximum(h, 0.0) if l else h
        h = (L.block @ a) @ w
    return h


def loss_and_backward(weights, plan: Plan, features, labels):
    """training.py:272-318 — mean LSE cross-entropy over labelled rows."""
    if plan.n_layers != len(weights):
        raise ValueError("plan depth does not match model depth")
    hs, us = [features[plan.input_nodes]], []
    for l, (L, w) in enumerate(zip(plan.layers, weights)):
        a = np.maximum(hs[-1], 0.0) if l else hs[-1]
        us.append(L.block @ a)
        hs.append(us[-1] @ w)
    logits = hs[-1]
    y_all = labels[plan.batch]
    lab = y_all >= 0
    n_lab = int(lab.sum())
    if n_lab == 0:
        raise ValueError("batch contains no labeled nodes")
    z, y = logits[lab], y_all[lab]
    zmax = z.max(axis=1, keepdims=True)
    lse = zmax[:, 0] + np.log(np.sum(np.exp(z - zmax), axis=1))
    loss = float(np.mean(lse - z[np.arange(n_lab), y]))
    gz = np.exp(z - lse[:, None])
    gz[np.arange(n_lab), y] -= 1.0
    gz /= n_lab
    g = np.zeros_like(logits)
    g[lab] = gz
    grads = [None] * len(weights)
    for l in range(len(weights) - 1, -1, -1):
        grads[l] = us[l].T @ g
        if l == 0:
            break
        g = (plan.layers[l].block.T @ (g @ weights[l].T)) * (hs[l] > 0.0)
    return loss, grads


def predict_logits(weights, g: Graph):
    """training.py:325-334 — exact full-graph forward."""
    P = g.to_sparse()
    h = g.features
    for l, w in enumerate(weights):
        h = (P @ (np.maximum(h, 0.0) if l else h)) @ w
    return h


# ---------------------------------------------------------------------------
# Simulated data-parallel loop (reference: training.py:370-518)
# ---------------------------------------------------------------------------


@dataclass
class MetricRow:
    epoch: int
    worker: int
    loss: float
    train_acc: float
    val_acc: float
    comm_nodes_epoch: int


def train_distributed(g: Graph, part: Partition, weights, cfg: SamplerConfig, *, epochs,
                      batch_size, lr, mode, seed, sampler="ladies", subgraph_size=None,
                      optimizer="sgd"):
    """training.py:430-518 — returns (metric rows, ledger counts); mutates weights.

    Worker gradients are summed in worker order from zeros and divided by the
    number of contributors, then SGD ``w -= lr*g`` (training.py:398-404) or
    Adam (training.py:407-427).
    """
    cfg = replace(cfg, mode=mode)
    k = part.n_workers
    L = len(weights)
    worker_train = [np.flatnonzero(g.train_mask & (part.owner == w)) for w in range(k)]
    active = [w for w in range(k) if len(worker_train[w])]
    for w in range(k):
        if not len(worker_train[w]):
            warnings.warn(f"worker {w} has no training nodes; skipping it")
    if not active:
        raise ValueError("no worker has training nodes")
    all_train = np.flatnonzero(g.train_mask)
    saint_norms = None
    if sampler == "saint":
        saint_norms = column_norms(g, all_train, all_train)
        per_epoch = max(1, int(np.ceil(len(all_train) / subgraph_size)))
    else:
        per_epoch = max(1, max(int(np.ceil(len(worker_train[w]) / batch_size))
                               for w in active))
    adam = None
    if optimizer == "adam":
        adam = {"t": 0, "m": [np.zeros_like(w) for w in weights],
                "v": [np.zeros_like(w) for w in weights]}
    ledger = np.zeros((epochs, k, L), dtype=np.int64)
    rows = []
    val_nodes = np.flatnonzero(g.val_mask) if g.val_mask is not None else np.empty(0, np.int64)
    for epoch in range(epochs):
        loss_sum = np.zeros(k)
        loss_cnt = np.zeros(k, dtype=np.int64)
        for it in range(per_epoch):
            acc = [np.zeros_like(w) for w in weights]
            contributors = 0
            for w in active:
                if sampler == "ladies":
                    brng = spawn_rng(seed, "batch", epoch, it, w)
                    take = min(batch_size, len(worker_train[w]))
                    batch = node_set(brng.choice(worker_train[w], size=take, replace=False))
                    plan = ladies_plan(g, part, w, batch, cfg, L,
                                       spawn_rng(seed, "plan", epoch, it, w))
                else:
                    plan = saint_plan(g, part, w, all_train, subgraph_size, cfg, L,
                                      spawn_rng(seed, "plan", epoch, it, w),
                                      norms=saint_norms)
                loss, grads = loss_and_backward(weights, plan, g.features, g.labels)
                for l in range(L):
                    acc[l] += grads[l]
                ledger[epoch, w, :] += plan.remote_per_layer()
                loss_sum[w] += loss
                loss_cnt[w] += 1
                contributors += 1
            avg = [a / contributors for a in acc]
            if adam is None:
                for wt, gr in zip(weights, avg):
                    wt -= lr * gr
            else:
                adam["t"] += 1
                t = adam["t"]
                for wt, gr, m, v in zip(weights, avg, adam["m"], adam["v"]):
                    m *= 0.9
                    m += (1 - 0.9) * gr
                    v *= 0.999
                    v += (1 - 0.999) * gr * gr
                    mh = m / (1 - 0.9 ** t)
                    vh = v / (1 - 0.999 ** t)
                    wt -= lr * mh / (np.sqrt(vh) + 1e-8)
        preds = np.argmax(predict_logits(weights, g), axis=1)
        val_acc = float(np.mean(preds[val_nodes] == g.labels[val_nodes])) if len(val_nodes) else 0.0
        for w in range(k):
            tw = worker_train[w]
            tr = float(np.mean(preds[tw] == g.labels[tw])) if len(tw) else 0.0
            ml = float(loss_sum[w] / loss_cnt[w]) if loss_cnt[w] else 0.0
            rows.append(MetricRow(epoch, w, ml, tr, val_acc, int(ledger[epoch, w].sum())))
    return rows, ledger
