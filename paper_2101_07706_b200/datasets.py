"""Dataset formats and the small-graph generator on the callers' side of the hot path
(SURVEY §8(f) rows 2 and 4).

* ``SbmSpec`` / ``synth_sbm``: the reference's block-model recipe (synth.py:14-95) for the
  experiment configs' ``dataset.synthetic`` section, graph-identical for the same spec: the
  same named random streams (``spawn_rng(seed, "sbm-edges" | "sbm-features" | "sbm-masks")``)
  drawn in the same order.  It enumerates the upper triangle, so it is meant for the small
  graphs the configs use; the benchmark shapes come from ``synth.make_shaped_graph`` (O(m)).
* Directory datasets (graph.py:115-367): ``edges.txt`` ("u v" lines, '#' comments),
  ``features.csv``, ``labels.csv`` ("node,label"), ``masks.csv`` ("node,split"), parsed with
  vectorised numpy instead of a per-line Python loop; a malformed file is re-scanned line by
  line only to report the reference's error message.
* ``load_partition_csv``: explicit "node,worker" assignments (partition.py:77-98).
"""

from __future__ import annotations

import csv
import io
import warnings
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .graph import WeightedGraph, graph_from_edges, normalize_weights, undirected_edges
from .partition import Partition
from .seeding import spawn_rng

SPLITS = ("train", "val", "test")


# ---------------------------------------------------------------------------- generator
@dataclass
class SbmSpec:
    """n_nodes split into n_blocks near-equal blocks; within-block pairs are edges with
    probability p_in, cross pairs with p_out; label = block id; features = one-hot of the
    block (mod feature_dim) plus N(0, noise_sigma) noise (synth.py:14-42)."""

    n_nodes: int
    n_blocks: int
    p_in: float
    p_out: float
    feature_dim: int
    noise_sigma: float = 0.0
    seed: int = 0

    def __post_init__(self) -> None:
        if self.n_nodes < 1 or self.n_blocks < 1:
            raise ValueError("n_nodes and n_blocks must be >= 1")
        if self.n_blocks > self.n_nodes:
            raise ValueError("more blocks than nodes")
        if not 0.0 <= self.p_out <= self.p_in <= 1.0:
            raise ValueError("need 0 <= p_out <= p_in <= 1")
        if self.feature_dim < 1:
            raise ValueError("feature_dim must be >= 1")
        if self.noise_sigma < 0.0:
            raise ValueError("noise_sigma must be >= 0")


def _block_of(n: int, k: int) -> np.ndarray:
    sizes = np.full(k, n // k, dtype=np.int64)
    sizes[: n % k] += 1
    return np.repeat(np.arange(k, dtype=np.int64), sizes)


def synth_sbm(spec: SbmSpec, normalize: bool = True) -> WeightedGraph:
    """Sample the block model with features, labels and 70/15/15 masks (synth.py:51-95)."""
    n, k = spec.n_nodes, spec.n_blocks
    if n > 1 and spec.p_in == 0.0 and spec.p_out == 0.0:
        warnings.warn("edgeless block model: every node ends up isolated")
    blk = _block_of(n, k)
    # one uniform per upper-triangle pair, row-major (np.triu_indices order)
    iu, ju = np.triu_indices(n, k=1)
    p_edge = np.where(blk[iu] == blk[ju], spec.p_in, spec.p_out)
    hit = spawn_rng(spec.seed, "sbm-edges").random(len(p_edge)) < p_edge
    g = graph_from_edges(np.stack([iu[hit], ju[hit]], axis=1).astype(np.int64), n_hint=n,
                         normalize=False)
    x = spawn_rng(spec.seed, "sbm-features").normal(0.0, spec.noise_sigma, size=(n, spec.feature_dim))
    x[np.arange(n), blk % spec.feature_dim] += 1.0
    perm = spawn_rng(spec.seed, "sbm-masks").permutation(n)
    n_tr, n_va = int(round(0.70 * n)), int(round(0.15 * n))
    masks = [np.zeros(n, dtype=bool) for _ in SPLITS]
    masks[0][perm[:n_tr]] = True
    masks[1][perm[n_tr:n_tr + n_va]] = True
    masks[2][perm[n_tr + n_va:]] = True
    g.features, g.labels = x, blk.copy()
    g.train_mask, g.val_mask, g.test_mask = masks
    return normalize_weights(g) if normalize else g


# ---------------------------------------------------------------------------- edge lists
def _edge_list_error(path: Path, text: str) -> ValueError:
    """Line-by-line re-scan of a file the vectorised parser rejected: the reference's
    message for the first offending line (graph.py:122-138)."""
    for lineno, line in enumerate(text.splitlines(), start=1):
        t = line.strip()
        if not t or t.startswith("#"):
            continue
        parts = t.split()
        if len(parts) != 2:
            return ValueError(f"{path}:{lineno}: expected 'u v', got {t!r}")
        try:
            u, v = int(parts[0]), int(parts[1])
        except ValueError:
            return ValueError(f"{path}:{lineno}: non-integer node id in {t!r}")
        if u < 0 or v < 0:
            return ValueError(f"{path}:{lineno}: negative node id in {t!r}")
    return ValueError(f"{path}: malformed edge list")


def load_edge_list(path, n_hint: int | None = None) -> WeightedGraph:
    """Undirected "u v" edge list -> un-normalised graph (both directions, duplicates
    collapsed); n = max id + 1, or n_hint when larger (graph.py:115-149)."""
    path = Path(path)
    text = path.read_text(encoding="utf-8")
    body = [ln for ln in (l.strip() for l in text.splitlines()) if ln and not ln.startswith("#")]
    if body:
        try:
            flat = np.array(" ".join(body).split(), dtype=np.int64)
        except ValueError:
            raise _edge_list_error(path, text) from None
        counts = np.fromiter((len(ln.split()) for ln in body), dtype=np.int64, count=len(body))
        if (counts != 2).any() or (flat < 0).any():
            raise _edge_list_error(path, text)
        e = flat.reshape(-1, 2)
    else:
        e = np.zeros((0, 2), dtype=np.int64)
    return graph_from_edges(e, n_hint=n_hint, normalize=False)


def save_edge_list(g: WeightedGraph, path) -> None:
    pairs = undirected_edges(g)
    with Path(path).open("w", encoding="utf-8", newline="\n") as fh:
        fh.write("".join(f"{u} {v}\n" for u, v in pairs))


# ---------------------------------------------------------------------------- CSV tables
def _pairs(path, header: str):
    """(int, str) rows of a two-column CSV with an optional header line."""
    out = []
    with Path(path).open("r", encoding="utf-8") as fh:
        for lineno, parts in enumerate(csv.reader(fh), start=1):
            if not parts:
                continue
            if lineno == 1 and not parts[0].strip().lstrip("-").isdigit():
                continue
            if len(parts) != 2:
                raise ValueError(f"{path}:{lineno}: expected '{header}'")
            out.append((int(parts[0]), parts[1].strip()))
    return out


def load_features_csv(path, n_nodes: int) -> np.ndarray:
    x = np.loadtxt(path, delimiter=",", dtype=np.float64, ndmin=2)
    if x.shape[0] != n_nodes:
        raise ValueError(f"feature rows ({x.shape[0]}) != n_nodes ({n_nodes})")
    return x


def save_features_csv(features: np.ndarray, path) -> None:
    buf = io.StringIO()
    for row in features:
        buf.write(",".join(repr(float(v)) for v in row) + "\n")
    Path(path).write_text(buf.getvalue(), encoding="utf-8", newline="\n")


def load_labels_csv(path, n_nodes: int) -> np.ndarray:
    """Class per node from "node,label" rows; -1 where absent."""
    y = np.full(n_nodes, -1, dtype=np.int64)
    for node, value in _pairs(path, "node,label"):
        if not 0 <= node < n_nodes:
            raise ValueError(f"label for out-of-range node {node}")
        y[node] = int(value)
    return y


def save_labels_csv(labels: np.ndarray, path) -> None:
    lines = ["node,label"] + [f"{i},{int(v)}" for i, v in enumerate(labels) if v >= 0]
    Path(path).write_text("\n".join(lines) + "\n", encoding="utf-8", newline="\n")


def load_masks_csv(path, n_nodes: int) -> dict:
    """train / val / test masks from "node,split" rows."""
    masks = {s: np.zeros(n_nodes, dtype=bool) for s in SPLITS}
    for node, split in _pairs(path, "node,split"):
        if split not in masks:
            raise ValueError(f"unknown split {split!r} (want train/val/test)")
        if not 0 <= node < n_nodes:
            raise ValueError(f"mask for out-of-range node {node}")
        masks[split][node] = True
    return masks


def save_masks_csv(masks: dict, path) -> None:
    n = len(next(iter(masks.values())))
    lines = ["node,split"] + [f"{i},{s}" for i in range(n) for s in SPLITS if masks[s][i]]
    Path(path).write_text("\n".join(lines) + "\n", encoding="utf-8", newline="\n")


def load_dataset(directory, n_hint: int | None = None, normalize: bool = True) -> WeightedGraph:
    """edges.txt plus the optional features / labels / masks CSVs of a directory; feature
    rows fix the node count (graph.py:321-351)."""
    d = Path(directory)
    x = None
    if (d / "features.csv").exists():
        x = np.loadtxt(d / "features.csv", delimiter=",", dtype=np.float64, ndmin=2)
        n_hint = max(n_hint or 0, x.shape[0])
    g = load_edge_list(d / "edges.txt", n_hint=n_hint)
    if normalize:
        g = normalize_weights(g)
    if x is not None:
        if x.shape[0] != g.n_nodes:
            raise ValueError(f"feature rows ({x.shape[0]}) != n_nodes ({g.n_nodes})")
        g.features = x
    if (d / "labels.csv").exists():
        g.labels = load_labels_csv(d / "labels.csv", g.n_nodes)
    if (d / "masks.csv").exists():
        m = load_masks_csv(d / "masks.csv", g.n_nodes)
        g.train_mask, g.val_mask, g.test_mask = m["train"], m["val"], m["test"]
    return g


def save_dataset(g: WeightedGraph, directory) -> None:
    """The layout load_dataset reads; the graph must be un-normalised (weights derive)."""
    if g.normalized:
        raise ValueError("save the un-normalized graph (weights are derived data)")
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    save_edge_list(g, d / "edges.txt")
    if g.features is not None:
        save_features_csv(g.features, d / "features.csv")
    if g.labels is not None:
        save_labels_csv(g.labels, d / "labels.csv")
    if g.train_mask is not None:
        save_masks_csv({"train": g.train_mask, "val": g.val_mask, "test": g.test_mask}, d / "masks.csv")


# ---------------------------------------------------------------------------- partitions
def load_partition_csv(path, n_nodes: int, k: int) -> Partition:
    """Explicit "node,worker" assignment covering every node (partition.py:77-98)."""
    owner = np.full(n_nodes, -1, dtype=np.int64)
    # rows are validated in file order, so the first bad line wins, as in the reference
    with Path(path).open("r", encoding="utf-8") as fh:
        for lineno, parts in enumerate(csv.reader(fh), start=1):
            if not parts:
                continue
            if lineno == 1 and not parts[0].strip().lstrip("-").isdigit():
                continue
            if len(parts) != 2:
                raise ValueError(f"{path}:{lineno}: expected 'node,worker'")
            node, w = int(parts[0]), int(parts[1])
            if not 0 <= node < n_nodes:
                raise ValueError(f"{path}:{lineno}: node {node} out of range")
            if not 0 <= w < k:
                raise ValueError(f"{path}:{lineno}: worker {w} out of range")
            owner[node] = w
    missing = np.flatnonzero(owner < 0)
    if len(missing):
        raise ValueError(f"partition file misses nodes {missing[:10].tolist()}")
    return Partition(n_workers=k, owner=owner, strategy="explicit")
