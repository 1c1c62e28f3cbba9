"""O(m) synthetic graphs of the benchmark shapes (Cora/Reddit/Amazon/YouTube-shaped).

The reference's generator (``synth.py:51-95``) enumerates all O(n^2) node pairs
and cannot build the 233K..1.6M-node shapes BASELINE.json names, so this module
draws the edge list directly: each undirected edge picks an endpoint u uniformly
and, with probability ``p_intra``, a partner from u's block (else uniformly).
Blocks are the labels, like the reference SBM (``synth.py:122-125``), and the
feature recipe follows ``synth.py:150-152`` (noise plus a block one-hot) or a
Cora-style Bernoulli bag of words.  Masks follow the seeded-shuffle split of
``synth.py:154-163``.

Everything is a deterministic function of (shape, seed): the canonical CSR is
unique, so it is identical whether built with numpy or with torch on a GPU.
Normalisation reproduces ``normalize_weights`` (``graph.py:166-183``) bit for bit
(self-loops, ``w = 1/sqrt(d_i*d_j)`` with IEEE sqrt and division).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

try:
    from .features import BitFeatures, pack_rows
except ImportError:  # loaded by path (bench.py's reference arm never imports the package)
    import importlib.util as _ilu
    import sys as _sys
    from pathlib import Path as _Path
    _spec = _ilu.spec_from_file_location("skg_features", _Path(__file__).with_name("features.py"))
    _feat = _ilu.module_from_spec(_spec)
    _sys.modules.setdefault("skg_features", _feat)
    _spec.loader.exec_module(_feat)
    BitFeatures, pack_rows = _feat.BitFeatures, _feat.pack_rows

# Shapes quoted in BASELINE.json:configs / SURVEY.md §8(d).  m is the number of
# undirected edge draws before dedup (self-pairs dropped).
SHAPES = {
    # Cora: 2,708 nodes, 5,278 undirected edges, 1,433-d binary features, 7 classes
    "cora": dict(n=2708, m=5278, F=1433, C=7, feat="bow", train=0.70, val=0.15, p_intra=0.80),
    # Reddit: 232,965 nodes, ~57.3M undirected edges (avg degree ~492), 602-d, 41 classes
    "reddit": dict(n=232965, m=57_300_000, F=602, C=41, feat="gauss", train=0.66, val=0.10,
                   p_intra=0.50),
    # reduced Reddit-like graph for fast parity tests (same recipe, ~29K candidates/layer)
    "reddit_s": dict(n=40000, m=2_000_000, F=602, C=41, feat="gauss", train=0.66, val=0.10,
                     p_intra=0.50),
    # Amazon (GraphSAINT): 1,598,960 nodes, ~132M CSR entries; F/C per SURVEY §8(d)4
    "amazon": dict(n=1598960, m=66_000_000, F=200, C=107, feat="gauss", train=0.85, val=0.05,
                   p_intra=0.50),
    "amazon_s": dict(n=120000, m=3_000_000, F=200, C=107, feat="gauss", train=0.85, val=0.05,
                     p_intra=0.50),
    # YouTube: 1.1M nodes, 6.1M CSR entries, 2048-d multi-hot, 64 labels
    "youtube": dict(n=1_100_000, m=3_050_000, F=2048, C=64, feat="bow", train=0.70, val=0.10,
                    p_intra=0.50, multilabel=0.03),
    # reduced YouTube-like graph for the multi-label parity tests
    "youtube_s": dict(n=30000, m=90000, F=256, C=64, feat="bow", train=0.70, val=0.10,
                      p_intra=0.50, multilabel=0.03),
}


@dataclass
class ShapedGraph:
    """Host-side normalised canonical CSR plus features, labels and masks."""

    name: str
    n_nodes: int
    offsets: np.ndarray      # int64 [n+1]
    neighbors: np.ndarray    # int32 [nnz] (ids < 2^31)
    weights: np.ndarray      # float64 [nnz]
    features: np.ndarray     # float32 [n, F]
    labels: np.ndarray       # int64 [n]
    train_mask: np.ndarray
    val_mask: np.ndarray
    test_mask: np.ndarray
    n_classes: int

    @property
    def nnz(self) -> int:
        return int(self.offsets[-1])

    def structure_hash(self) -> str:
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(self.offsets, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(self.neighbors, dtype=np.int64).tobytes())
        return h.hexdigest()

    def features_hash(self) -> str:
        if isinstance(self.features, BitFeatures):  # packed rows: hash the words
            return hashlib.sha256(self.features.words.tobytes()).hexdigest()
        return hashlib.sha256(np.ascontiguousarray(self.features).tobytes()).hexdigest()


def _blocks(n: int, k: int) -> np.ndarray:
    counts = np.full(k, n // k, dtype=np.int64)
    counts[: n % k] += 1
    return np.repeat(np.arange(k, dtype=np.int64), counts)


def _edge_draws(n, m, blocks, k, p_intra, rng):
    counts = np.bincount(blocks, minlength=k)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    us, vs = [], []
    chunk = 4_000_000
    done = 0
    while done < m:
        c = min(chunk, m - done)
        u = rng.integers(0, n, size=c, dtype=np.int64)
        intra = rng.random(c) < p_intra
        b = blocks[u]
        v_in = starts[b] + (rng.random(c) * counts[b]).astype(np.int64)
        v_any = rng.integers(0, n, size=c, dtype=np.int64)
        v = np.where(intra, v_in, v_any)
        keep = u != v
        us.append(u[keep])
        vs.append(v[keep])
        done += c
    return np.concatenate(us), np.concatenate(vs)


def _normalised_csr_numpy(u, v, n):
    loop = np.arange(n, dtype=np.int64)
    key = np.concatenate([u * n + v, v * n + u, loop * n + loop])
    key.sort()  # sort + adjacent-diff dedup (np.unique is hash-based and slow here)
    key = key[np.concatenate([[True], key[1:] != key[:-1]])]
    row, col = key // n, key % n
    deg = np.bincount(row, minlength=n).astype(np.int64)
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=offs[1:])
    d = deg.astype(np.float64)
    w = 1.0 / np.sqrt(d[row] * d[col])
    return offs, col.astype(np.int32), w


def _normalised_csr_torch(u, v, n, device):
    import torch
    tu = torch.from_numpy(u).to(device)
    tv = torch.from_numpy(v).to(device)
    loop = torch.arange(n, device=device, dtype=torch.int64)
    key = torch.cat([tu * n + tv, tv * n + tu, loop * n + loop])
    del tu, tv
    key = torch.unique(key, sorted=True)
    row, col = key // n, key % n
    del key
    deg = torch.bincount(row, minlength=n)
    offs = torch.zeros(n + 1, dtype=torch.int64, device=device)
    offs[1:] = torch.cumsum(deg, 0)
    d = deg.to(torch.float64)
    w = 1.0 / torch.sqrt(d[row] * d[col])
    return offs.cpu().numpy(), col.to(torch.int32).cpu().numpy(), w.cpu().numpy()


def make_shaped_graph(name: str, seed: int = 0, device: str | None = None,
                      with_features: bool = True, packed: bool = False) -> ShapedGraph:
    """Build the named shape deterministically.  device='cuda' speeds up the sort.
    packed=True returns bag-of-words (multi-hot) features as BitFeatures, generated in row
    chunks from the same random stream (identical values; the YouTube shape's 2048-d rows
    never exist densely on the host)."""
    s = SHAPES[name]
    n, m, F, C = s["n"], s["m"], s["F"], s["C"]
    root = np.random.SeedSequence([seed, int.from_bytes(name.encode()[:8].ljust(8, b"\0"), "little")])
    r_edge, r_feat, r_mask, r_lab = [np.random.default_rng(c) for c in root.spawn(4)]
    blocks = _blocks(n, C)
    u, v = _edge_draws(n, m, blocks, C, s["p_intra"], r_edge)
    if device is not None and device != "cpu":
        offs, col, w = _normalised_csr_torch(u, v, n, device)
    else:
        offs, col, w = _normalised_csr_numpy(u, v, n)
    del u, v
    if with_features:
        if s["feat"] == "gauss":
            x = r_feat.standard_normal(size=(n, F), dtype=np.float32)
            x[np.arange(n), blocks % F] += np.float32(1.0)
        elif packed:  # the same draws as below, packed 32 features per word as they come
            words = np.zeros((n, (F + 31) // 32), dtype="<u4")
            ch = max(1, (1 << 24) // F)
            for s0 in range(0, n, ch):
                xb = r_feat.random((min(ch, n - s0), F), dtype=np.float32) < 0.0127
                words[s0:s0 + len(xb)] = pack_rows(xb)
            sig = (blocks * 10) % F
            for j in range(10):
                on = r_feat.random(n) < 0.3
                cols = (sig[on] + j) % F
                np.bitwise_or.at(words, (np.flatnonzero(on), cols >> 5),
                                 (np.uint32(1) << (cols & 31).astype(np.uint32)).astype("<u4"))
            x = BitFeatures(words, F)
        else:  # Bernoulli bag of words with a block signal
            x = (r_feat.random((n, F), dtype=np.float32) < 0.0127).astype(np.float32)
            sig = (blocks * 10) % F
            for j in range(10):
                on = r_feat.random(n) < 0.3
                x[np.flatnonzero(on), (sig[on] + j) % F] = 1.0
    else:
        x = np.zeros((n, 0), dtype=np.float32)
    order = r_mask.permutation(n)
    n_tr = int(round(s["train"] * n))
    n_va = int(round(s["val"] * n))
    tr = np.zeros(n, bool)
    va = np.zeros(n, bool)
    te = np.zeros(n, bool)
    tr[order[:n_tr]] = True
    va[order[n_tr:n_tr + n_va]] = True
    te[order[n_tr + n_va:]] = True
    labels = blocks.copy()
    if s.get("multilabel"):  # multi-hot: the block's label plus independent extra labels
        labels = r_lab.random((n, C), dtype=np.float32) < np.float32(s["multilabel"])
        labels[np.arange(n), blocks % C] = True
    return ShapedGraph(name, n, offs, col, w, x, labels, tr, va, te, C)
