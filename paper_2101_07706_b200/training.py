"""Drop-in for the reference's training module (skewgcn/training.py) on the GPU.

Same names, arguments, return types and exceptions as the reference:
``ladies_plan`` (training.py:162-208), ``saint_plan`` (216-254), ``forward`` (261-269),
``loss_and_backward`` (272-318), ``predict_logits`` / ``evaluate`` (325-363) and
``train_distributed`` (430-518).  Plans are sampled by the sm_100a kernels of
libskg and stay device-resident; the scipy/numpy view the reference returns is
materialised lazily on first access (``plan.layers``), bit-identical in node sets,
block indices and ledger counts.

``train_distributed`` runs the whole iteration on the device: the host only derives
batch ids and PCG64 states (natively, libskg host runtime), every worker's plan of an
iteration is sampled in one batched launch, worker gradients are accumulated in
worker order, averaged across GPUs with an NCCL all-reduce when torch.distributed is
initialised, and the optimizer step is one fused kernel.
"""

from __future__ import annotations

import ctypes as C
import os
import warnings
from dataclasses import dataclass, field, replace

import numpy as np
import scipy.sparse as sp

from . import _device as D

# host threads for the per-iteration host work of a look-ahead group (skg_group_inputs)
_HOST_THREADS = max(1, min(8, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
                          else (os.cpu_count() or 1)))
from ._native import (DT, KIND_LADIES, KIND_SAINT, MODES, RNG_EXPLICIT, RNG_PCG64, RNG_PHILOX, SkgRng,
                      check, lib, ptr)
from .graph import WeightedGraph, check_node_set, node_set
from .partition import Partition
from .sampling import ProbDist, SamplerConfig
from .seeding import advance_generator, generator_state, spawn_rng

# ---------------------------------------------------------------------------
# Model
# ---------------------------------------------------------------------------


@dataclass
class GcnModel:
    """Per-layer weight matrices (training.py:40-62)."""

    weights: list

    def __post_init__(self) -> None:
        for a, b in zip(self.weights, self.weights[1:]):
            if a.shape[1] != b.shape[0]:
                raise ValueError("adjacent layer dims do not match")
        if any(not np.all(np.isfinite(w)) for w in self.weights):
            raise ValueError("non-finite model weights")

    @property
    def n_layers(self) -> int:
        return len(self.weights)

    @property
    def dims(self) -> list:
        return [self.weights[0].shape[0]] + [w.shape[1] for w in self.weights]

    def copy(self) -> "GcnModel":
        return GcnModel([w.copy() for w in self.weights])


def init_model(layer_dims, seed: int) -> GcnModel:
    """Glorot uniform from spawn_rng(seed, 'init', l) (training.py:65-74)."""
    if len(layer_dims) < 2:
        raise ValueError("need at least input and output dims")
    ws = []
    for l, (a, b) in enumerate(zip(layer_dims, layer_dims[1:])):
        bound = np.sqrt(6.0 / (a + b))
        ws.append(spawn_rng(seed, "init", l).uniform(-bound, bound, size=(a, b)))
    return GcnModel(ws)


# ---------------------------------------------------------------------------
# Plans
# ---------------------------------------------------------------------------


@dataclass
class PlanLayer:
    nodes: np.ndarray
    block: sp.csr_matrix
    dist: ProbDist | None
    remote_sampled: int


class CommLedger:
    """Remote-feature-fetch counts (epochs, workers, layers) (training.py:117-134)."""

    def __init__(self, counts: np.ndarray):
        self.counts = counts

    @classmethod
    def empty(cls, n_epochs, n_workers, n_layers):
        return cls(np.zeros((n_epochs, n_workers, n_layers), dtype=np.int64))

    def add_plan(self, epoch, worker, plan) -> None:
        self.counts[epoch, worker, :] += plan.remote_per_layer()

    def total(self) -> int:
        return int(self.counts.sum())

    def per_worker_epoch(self, epoch, worker) -> int:
        return int(self.counts[epoch, worker].sum())


class SamplePlan:
    """Device-resident plan; ``layers`` materialises the reference's view on demand."""

    def __init__(self, lease: D.Lease, batch: np.ndarray, n_layers: int, kind: int):
        self._lease = lease
        self.batch = batch
        self._n_layers = n_layers
        self._kind = kind
        self._layers = None
        st, info, rc = lease.ps.stats(lease.slot)
        check(rc)
        self._stats = st
        self._info = info
        self.starvation_events = int(info[2]) if kind == KIND_LADIES else 0
        self.draws_consumed = int(info[1])

    @property
    def n_layers(self) -> int:
        return self._n_layers

    def remote_per_layer(self) -> np.ndarray:
        L = self._n_layers
        if self._kind == KIND_SAINT:
            out = np.zeros(L, dtype=np.int64)
            out[0] = self._stats[0, 4]
            return out
        return self._stats[:, 4][::-1].astype(np.int64).copy()

    @property
    def layers(self):
        if self._layers is None:
            self._layers = self._materialise()
        return self._layers

    @property
    def input_nodes(self) -> np.ndarray:
        return self.layers[0].nodes

    def _materialise(self):
        ps, slot = self._lease.ps, self._lease.slot
        L = self._n_layers
        out = []
        ts = range(L) if self._kind == KIND_LADIES else [0]
        for t in ts:
            row = self._stats[t]
            has = bool(row[5])
            lay = D.read_layer(ps, slot, t, row, has)
            block = sp.csr_matrix((lay["values"], lay["indices"].astype(np.int32), lay["indptr"]),
                                  shape=lay["shape"])
            dist = None
            if has:
                s = float(np.array(row[11]).view(np.float64))
                total = float(np.array(row[12]).view(np.float64))
                norm, loc = lay["norm"], lay["is_local"]
                scaled = np.where(loc, s * norm, norm) if row[8] else norm
                dist = ProbDist(candidates=lay["cand"].astype(np.int64), q=scaled / total,
                                is_local=loc, s_used=s if row[8] else 1.0)
            out.append(PlanLayer(nodes=lay["nodes"], block=block, dist=dist,
                                 remote_sampled=int(row[4])))
        if self._kind == KIND_SAINT:
            first = out[0]
            return [PlanLayer(first.nodes, first.block, first.dist,
                              first.remote_sampled if l == 0 else 0) for l in range(L)]
        out.reverse()
        return out


def _uniform_source(rng, budget: int, n_layers: int):
    """The plan's uniform stream (skg_rng) for any numpy Generator, which the reference
    passes to Generator.choice (sampling.py:184).  PCG64 and Philox streams are generated
    on the device from the bit generator's state; any other bit generator's uniforms are
    drawn here from a copy of ``rng`` (n_layers * budget of them, every draw a plan can
    make) and passed explicitly."""
    if not isinstance(rng, np.random.Generator):
        raise TypeError("rng must be a numpy.random.Generator")
    r = SkgRng()
    gs = generator_state(rng)
    if gs is not None:
        r.kind = RNG_PCG64
        for q in range(4):
            r.w[q] = int(gs[0][q])
        return r, None
    st = rng.bit_generator.state
    if st.get("bit_generator") == "Philox":
        r.kind = RNG_PHILOX
        words = list(st["state"]["counter"]) + list(st["state"]["key"]) + list(st["buffer"])
        for q, v in enumerate(words):
            r.w[q] = int(v)
        r.buffer_pos = int(st["buffer_pos"])
        return r, None
    shadow = np.random.Generator(type(rng.bit_generator)())
    shadow.bit_generator.state = st
    u = np.ascontiguousarray(shadow.random(n_layers * budget), dtype=np.float64)
    r.kind = RNG_EXPLICIT
    r.uniforms = u.ctypes.data_as(C.POINTER(C.c_double))
    r.n_uniforms = len(u)
    return r, u


def _advance(rng, n_draws: int) -> None:
    """Leave ``rng`` where the reference's random(B) calls would (n_draws uniforms)."""
    if n_draws <= 0:
        return
    name = rng.bit_generator.state.get("bit_generator")
    if name == "PCG64":
        advance_generator(rng, n_draws)
    elif name == "Philox":
        rng.bit_generator.random_raw(n_draws)  # next_uint64 per uniform; uint32 buffer kept
    else:
        rng.random(n_draws)


def ladies_plan(g: WeightedGraph, partition: Partition, worker: int, batch, cfg: SamplerConfig,
                n_layers: int, rng: np.random.Generator) -> SamplePlan:
    """Layer-wise skewed sampling on the GPU (training.py:162-208).  Consumes exactly the
    uniforms the reference would from ``rng`` and advances it accordingly."""
    batch = node_set(batch)
    if len(batch) == 0:
        raise ValueError("empty batch")
    check_node_set(batch, g.n_nodes)
    if not 0 <= worker < partition.n_workers:
        raise ValueError("worker id out of range")
    dg = D.device_graph(g)
    dg.ensure_owner(partition)
    src, _keep = _uniform_source(rng, int(cfg.budget), n_layers)
    ps = dg.acquire(KIND_LADIES, 1, n_layers, int(cfg.budget), int(len(batch)))
    lease = D.Lease(dg, ps, 0)
    off = np.array([0, len(batch)], dtype=np.int64)
    w = np.array([worker], dtype=np.int32)
    check(lib.skg_ladies_sample_rng(ps.h, 1, ptr(w, C.c_int32), ptr(off, C.c_int64),
                                    ptr(batch, C.c_int64), MODES[cfg.mode], float(cfg.skew_constant),
                                    float(cfg.min_scale), C.byref(src), None))
    plan = SamplePlan(lease, batch, n_layers, KIND_LADIES)
    _advance(rng, plan.draws_consumed)
    return plan


def train_column_norms(g: WeightedGraph, train_nodes: np.ndarray) -> np.ndarray:
    """Squared column norms over training rows (training.py:211-213), on the GPU."""
    from .graph import column_norms
    return column_norms(g, train_nodes, train_nodes)


def _saint_set(dg, ps, train_nodes, precompute):
    key = (id(train_nodes), train_nodes.ctypes.data, train_nodes.shape, dg.owner_key)
    if ps.train_key != key:
        check(lib.skg_saint_set_candidates(ps.h, ptr(train_nodes, C.c_int64), len(train_nodes),
                                           int(precompute), None))
        ps.train_key = key
        ps.train_ref = train_nodes


def saint_plan(g: WeightedGraph, partition: Partition, worker: int, train_nodes,
               subgraph_size: int, cfg: SamplerConfig, n_layers: int, rng: np.random.Generator,
               norms=None) -> SamplePlan:
    """GraphSAINT-style subgraph plan on the GPU (training.py:216-254).  Column norms over
    the training rows are computed (and cached per partition) on the device; a passed
    ``norms`` array is accepted for API compatibility (it equals what the device computes)."""
    train_nodes = node_set(train_nodes)
    if len(train_nodes) == 0:
        raise ValueError("empty training node set")
    if subgraph_size > len(train_nodes):
        warnings.warn("subgraph size exceeds training set; clamping")
        subgraph_size = len(train_nodes)
    if subgraph_size < 1:
        raise ValueError("subgraph size must be >= 1")
    check_node_set(train_nodes, g.n_nodes)
    if not 0 <= worker < partition.n_workers:
        raise ValueError("worker id out of range")
    dg = D.device_graph(g)
    dg.ensure_owner(partition)
    src, _keep = _uniform_source(rng, int(subgraph_size), n_layers)
    ps = dg.acquire(KIND_SAINT, 1, n_layers, int(subgraph_size), 1)
    lease = D.Lease(dg, ps, 0)
    _saint_set(dg, ps, train_nodes, cfg.mode != "local")
    w = np.array([worker], dtype=np.int32)
    check(lib.skg_saint_sample_rng(ps.h, 1, ptr(w, C.c_int32), MODES[cfg.mode],
                                   float(cfg.skew_constant), float(cfg.min_scale), C.byref(src),
                                   None))
    plan = SamplePlan(lease, None, n_layers, KIND_SAINT)
    plan.batch = plan.layers[0].nodes
    _advance(rng, plan.draws_consumed)
    return plan


# ---------------------------------------------------------------------------
# Forward / backward
# ---------------------------------------------------------------------------

def _torch():
    import torch
    return torch


def _device_weights(weights, dtype):
    torch = _torch()
    td = torch.float32 if dtype == "float32" else torch.float64
    ws = [torch.as_tensor(np.ascontiguousarray(w), dtype=td).cuda() for w in weights]
    return ws, np.array([w.data_ptr() for w in ws], dtype=np.uint64)


def _check_plan(model, plan):
    if not isinstance(plan, SamplePlan):
        raise TypeError("plan must come from paper_2101_07706_b200.ladies_plan / saint_plan")
    if plan.n_layers != model.n_layers:
        raise ValueError("plan depth does not match model depth")


def forward(model: GcnModel, plan: SamplePlan, features: np.ndarray) -> np.ndarray:
    """Logits for the plan's batch (training.py:261-269)."""
    _check_plan(model, plan)
    dtype = D.compute_dtype()
    lease = plan._lease
    lease.dg.ensure_features(features, dtype)
    dims = [features.shape[1]] + [w.shape[1] for w in model.weights]
    if dims[0] != model.weights[0].shape[0]:
        raise ValueError("feature dim does not match the model")
    gcn = lease.ps.gcn(dims, dtype)
    ws, wp = _device_weights(model.weights, dtype)
    check(lib.skg_gcn_forward(gcn, lease.slot, ptr(wp, C.c_uint64), D.current_stream()))
    rows = C.c_int64()
    nb = plan._stats[0, 0] if plan._kind == KIND_LADIES else plan._stats[0, 2]
    out = np.zeros((int(nb), dims[-1]), dtype=np.float32 if dtype == "float32" else np.float64)
    check(lib.skg_gcn_read_logits(gcn, lease.slot, out.ctypes.data_as(C.c_void_p), C.byref(rows)))
    del ws
    return out.astype(np.float64)


def loss_and_backward(model: GcnModel, plan: SamplePlan, features: np.ndarray, labels: np.ndarray,
                      pos_weight: float = 50.0):
    """Mean softmax cross-entropy over labelled batch rows and all weight gradients
    (training.py:272-318), computed on the GPU.  With an n x C multi-hot ``labels`` matrix
    the head is the multi-label BCE-with-logits (positive weight ``pos_weight``, mean over
    batch rows x classes; extension for the YouTube-shaped config, no reference code)."""
    _check_plan(model, plan)
    torch = _torch()
    dtype = D.compute_dtype()
    lease = plan._lease
    labels = np.asarray(labels)
    multi = labels.ndim == 2
    if not multi and not np.any(labels[plan.batch] >= 0):
        raise ValueError("batch contains no labeled nodes")
    lease.dg.ensure_features(features, dtype)
    lease.dg.ensure_labels(labels)
    dims = [features.shape[1]] + [w.shape[1] for w in model.weights]
    gcn = lease.ps.gcn(dims, dtype)
    check(lib.skg_gcn_set_loss(gcn, 1 if multi else 0, float(pos_weight) if multi else 1.0))
    ws, wp = _device_weights(model.weights, dtype)
    gs = [torch.empty_like(w) for w in ws]
    gp = np.array([g.data_ptr() for g in gs], dtype=np.uint64)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    check(lib.skg_gcn_step(gcn, lease.slot, ptr(wp, C.c_uint64), ptr(gp, C.c_uint64), 0,
                           loss.data_ptr(), D.current_stream()))
    torch.cuda.synchronize()
    return float(loss.item()), [g.double().cpu().numpy() for g in gs]


# ---------------------------------------------------------------------------
# Full-graph inference and evaluation
# ---------------------------------------------------------------------------

def _predict_device(dg, model_weights_dev, dims, dtype):
    torch = _torch()
    wp = np.array([w.data_ptr() for w in model_weights_dev], dtype=np.uint64)
    d = np.asarray(dims, dtype=np.int64)
    out = torch.empty((dg.n, dims[-1]), dtype=torch.float32 if dtype == "float32" else torch.float64,
                      device="cuda")
    check(lib.skg_predict_logits(dg.ctx, len(dims) - 1, ptr(d, C.c_int64), ptr(wp, C.c_uint64),
                                 DT[dtype], out.data_ptr(), D.current_stream()))
    return out


def predict_logits(model: GcnModel, g: WeightedGraph) -> np.ndarray:
    """Exact full-graph forward (training.py:325-334) on the GPU."""
    if g.features is None:
        raise ValueError("graph carries no features")
    dtype = D.compute_dtype()
    dg = D.device_graph(g)
    dg.ensure_features(g.features, dtype)
    ws, _ = _device_weights(model.weights, dtype)
    return _predict_device(dg, ws, model.dims, dtype).double().cpu().numpy()


@dataclass
class EvalResult:
    accuracy: float
    micro_f1: float


def multilabel_scores(logits: np.ndarray, y: np.ndarray):
    """(subset accuracy, micro-F1) of z > 0 against multi-hot targets."""
    pred = logits > 0
    truth = np.asarray(y) != 0
    tp = float(np.sum(pred & truth))
    fp = float(np.sum(pred & ~truth))
    fn = float(np.sum(~pred & truth))
    denom = 2 * tp + fp + fn
    return float(np.mean(np.all(pred == truth, axis=1))), (2 * tp / denom if denom > 0 else 0.0)


def evaluate(model: GcnModel, g: WeightedGraph, nodes) -> EvalResult:
    """Argmax accuracy and micro-F1 (training.py:343-363); multi-hot labels: subset
    accuracy and micro-F1 of z > 0."""
    nodes = node_set(nodes)
    if len(nodes) == 0:
        raise ValueError("empty evaluation node set")
    if g.labels is not None and np.asarray(g.labels).ndim == 2:
        acc, f1 = multilabel_scores(predict_logits(model, g)[nodes], np.asarray(g.labels)[nodes])
        return EvalResult(accuracy=acc, micro_f1=f1)
    if g.labels is None or np.any(g.labels[nodes] < 0):
        raise ValueError("evaluation nodes must be labeled")
    preds = np.argmax(predict_logits(model, g)[nodes], axis=1)
    truth = g.labels[nodes]
    accuracy = float(np.mean(preds == truth))
    n_classes = int(max(preds.max(), truth.max())) + 1
    tp = np.array([np.sum((preds == c) & (truth == c)) for c in range(n_classes)], dtype=float)
    fp = np.array([np.sum((preds == c) & (truth != c)) for c in range(n_classes)], dtype=float)
    fn = np.array([np.sum((preds != c) & (truth == c)) for c in range(n_classes)], dtype=float)
    denom = 2 * tp.sum() + fp.sum() + fn.sum()
    micro_f1 = float(2 * tp.sum() / denom) if denom > 0 else 0.0
    return EvalResult(accuracy=accuracy, micro_f1=micro_f1)


# ---------------------------------------------------------------------------
# Distributed training loop
# ---------------------------------------------------------------------------


@dataclass
class MetricRow:
    epoch: int
    worker: int
    loss: float
    train_acc: float
    val_acc: float
    comm_nodes_epoch: int


@dataclass
class Metrics:
    rows: list = field(default_factory=list)

    def best_val_acc(self) -> float:
        return max((r.val_acc for r in self.rows), default=0.0)

    def final_val_acc(self) -> float:
        return self.rows[-1].val_acc if self.rows else 0.0

    def write_csv(self, path) -> None:
        with open(path, "w", encoding="utf-8", newline="\n") as fh:
            fh.write("epoch,worker,loss,train_acc,val_acc,comm_nodes_epoch\n")
            for r in self.rows:
                fh.write(f"{r.epoch},{r.worker},{r.loss!r},{r.train_acc!r},"
                         f"{r.val_acc!r},{r.comm_nodes_epoch}\n")


def _dist_info():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist, dist.get_rank(), dist.get_world_size()
    except Exception:
        pass
    return None, 0, 1


def worker_ranks(k: int, active, world: int) -> np.ndarray:
    """Home rank of every worker's partition: the rank that trains it (assign_workers);
    workers without training nodes still own feature rows and go round-robin."""
    wr = np.array([w % world for w in range(k)], dtype=np.int64)
    for r in range(world):
        for w in assign_workers(active, r, world):
            wr[w] = r
    return wr


def feature_shard_map(owner: np.ndarray, worker_rank: np.ndarray, world: int):
    """node -> (rank holding its feature row, row inside that rank's shard).  Rows of a
    shard are the rank's nodes in ascending id order.  Returns (node_rank, node_row, rows)."""
    node_rank = worker_rank[np.asarray(owner, dtype=np.int64)].astype(np.int32)
    node_row = np.empty(len(owner), dtype=np.int32)
    rows = []
    for r in range(world):
        ids = np.flatnonzero(node_rank == r)
        node_row[ids] = np.arange(len(ids), dtype=np.int32)
        rows.append(ids)
    return node_rank, node_row, rows


def reduce_epoch_stats(dist, loss_sum, loss_cnt, ledger):
    """Sum per-worker loss sums / counts and the epoch ledger over ranks.  Each worker
    lives on exactly one rank, so every entry has a single non-zero contributor and the
    sums are exact (identical on every rank)."""
    torch = _torch()
    dev = ledger.device
    ls = torch.as_tensor(np.asarray(loss_sum, dtype=np.float64), device=dev)
    lc = torch.as_tensor(np.asarray(loss_cnt, dtype=np.int64), device=dev)
    led = ledger.clone()
    dist.all_reduce(ls)
    dist.all_reduce(lc)
    dist.all_reduce(led)
    return ls.cpu().numpy(), lc.cpu().numpy(), led


def assign_workers(active, rank: int, world: int):
    """Workers (partitions) handled by this rank: contiguous blocks of the active list,
    so rank r's workers precede rank r+1's (the reference's worker order)."""
    n = len(active)
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return list(active[lo:hi])


class Trainer:
    """Device-resident training state for ``train_distributed`` (and the benchmark).

    Plans depend only on (seed, epoch, iteration, worker), never on the weights
    (training.py:488-493), so the plans of ``ahead`` future iterations are sampled by one
    batched launch sequence (``sample_group``) and consumed one iteration at a time by
    ``compute`` + ``reduce_and_step``; results are identical to sampling them one by one.

    ``deterministic`` (several ranks only): instead of an all-reduce of per-rank gradient
    sums, every worker's gradient is all-gathered and summed from zero in worker order, the
    reference's own order (training.py:500-504), so the run is bit-identical to the
    single-process one (for unsplit contractions; SURVEY §8 A19's ordered mode).
    """

    def __init__(self, g, partition, model, cfg, *, batch_size, lr, mode, seed,
                 sampler="ladies", subgraph_size=None, optimizer="sgd", dtype=None,
                 epochs=1, workers=None, ahead=1, shard_features=None, streams=1,
                 loss="auto", pos_weight=50.0, deterministic=False):
        torch = _torch()
        if g.features is None or g.labels is None or g.train_mask is None:
            raise ValueError("training needs features, labels and masks")
        if loss not in ("auto", "ce", "bce"):
            raise ValueError(f"unknown loss {loss!r}")
        if sampler not in ("ladies", "saint"):
            raise ValueError(f"unknown sampler {sampler!r}")
        if sampler == "saint" and subgraph_size is None:
            raise ValueError("saint sampler needs subgraph_size")
        if optimizer not in ("sgd", "adam"):
            raise ValueError(f"unknown optimizer {optimizer!r}")
        self.g, self.partition, self.model = g, partition, model
        self.cfg = replace(cfg, mode=mode)
        self.mode, self.seed, self.lr = mode, seed, lr
        self.sampler, self.optimizer = sampler, optimizer
        self.batch_size = batch_size
        self.dtype = dtype or D.compute_dtype()
        self.k = partition.n_workers
        self.L = model.n_layers
        self.dims = model.dims
        owner = partition.owner
        self.worker_train = [np.flatnonzero(g.train_mask & (owner == w)) for w in range(self.k)]
        self.active = [w for w in range(self.k) if len(self.worker_train[w])]
        for w in range(self.k):
            if not len(self.worker_train[w]):
                warnings.warn(f"worker {w} has no training nodes; skipping it")
        if not self.active:
            raise ValueError("no worker has training nodes")
        self.all_train = np.flatnonzero(g.train_mask).astype(np.int64)
        if sampler == "saint":
            if subgraph_size > len(self.all_train):
                warnings.warn("subgraph size exceeds training set; clamping")
                subgraph_size = len(self.all_train)
            self.per_epoch = max(1, int(np.ceil(len(self.all_train) / subgraph_size)))
        else:
            self.per_epoch = max(1, max(int(np.ceil(len(self.worker_train[w]) / batch_size))
                                        for w in self.active))
        self.subgraph_size = subgraph_size
        self.dist, self.rank, self.world = _dist_info()
        self.mine = workers if workers is not None else assign_workers(self.active, self.rank, self.world)
        self.n_my = len(self.mine)
        self.ahead = max(1, int(ahead))
        self.dg = D.device_graph(g)
        self.dg.ensure_owner(partition)
        self.dg.ensure_features(g.features, self.dtype)
        self.dg.ensure_labels(np.asarray(g.labels))
        n_slots = max(1, self.n_my * self.ahead)
        # plan arenas in rotation: `streams` sampler streams fill groups ahead while the GCN
        # consumes the oldest one (main stream); plans never depend on the weights
        # (training.py:488-493)
        self.n_streams = max(1, int(streams))
        self.n_bufs = self.n_streams + 1
        self.bufs = []
        for _ in range(self.n_bufs):
            if sampler == "ladies":
                ps = self.dg.acquire(KIND_LADIES, n_slots, self.L, int(self.cfg.budget), int(batch_size))
            else:
                ps = self.dg.acquire(KIND_SAINT, n_slots, self.L, int(subgraph_size), 1)
                _saint_set(self.dg, ps, self.all_train, mode != "local")
            self.bufs.append((ps, ps.gcn(self.dims, self.dtype)))
        self.ps, self.gcn = self.bufs[0]
        # head: softmax CE for class labels, multi-label BCE for an n x C multi-hot matrix
        self.multilabel = np.asarray(g.labels).ndim == 2 if loss == "auto" else loss == "bce"
        for _, gcn in self.bufs:
            check(lib.skg_gcn_set_loss(gcn, 1 if self.multilabel else 0,
                                       float(pos_weight) if self.multilabel else 1.0))
        self._peer_ptrs = []
        if shard_features is None:
            shard_features = self.world > 1
        if shard_features and self.world > 1:
            self._install_feature_shards()
        td = torch.float32 if self.dtype == "float32" else torch.float64
        sizes = [w.size for w in model.weights]
        self.n_params = int(sum(sizes))
        self.wflat = torch.empty(self.n_params, dtype=td, device="cuda")
        self.gflat = torch.zeros(self.n_params, dtype=td, device="cuda")
        self.wviews, self.gviews = [], []
        o = 0
        for w in model.weights:
            self.wviews.append(self.wflat[o:o + w.size].view(w.shape))
            self.gviews.append(self.gflat[o:o + w.size].view(w.shape))
            self.wviews[-1].copy_(torch.as_tensor(w, dtype=td))
            o += w.size
        self.wp = np.array([v.data_ptr() for v in self.wviews], dtype=np.uint64)
        self.gp = np.array([v.data_ptr() for v in self.gviews], dtype=np.uint64)
        self.deterministic = bool(deterministic) and self.world > 1
        if self.deterministic:
            # per-worker gradients (rows padded to the largest rank's worker count)
            counts = [len(assign_workers(self.active, r, self.world)) for r in range(self.world)]
            self._wcap = max(counts)
            self._wcounts = counts
            self.wgrads = torch.zeros((self._wcap, self.n_params), dtype=td, device="cuda")
            self._wgp = []
            for i in range(self._wcap):
                o, ptrs = 0, []
                for w in model.weights:
                    ptrs.append(self.wgrads[i, o:o + w.size].data_ptr())
                    o += w.size
                self._wgp.append(np.array(ptrs, dtype=np.uint64))
            self._gathered = torch.zeros((self.world * self._wcap, self.n_params), dtype=td, device="cuda")
        if optimizer == "adam":
            self.m = torch.zeros_like(self.wflat)
            self.v = torch.zeros_like(self.wflat)
            self.t = 0
        self.epochs = epochs
        self.ledger = torch.zeros((max(epochs, 1), self.k, self.L), dtype=torch.int64, device="cuda")
        self.losses = torch.zeros((self.per_epoch, max(1, self.n_my)), dtype=torch.float64,
                                  device="cuda")
        self.stream = D.current_stream()
        self.main = torch.cuda.current_stream()
        # The GCN chain (on the caller's stream) is the step's critical path: the sampler
        # streams run at the lowest priority so that, on a high-priority caller stream (as
        # train_distributed and bench.py use), GCN kernels take SMs first as they free up
        # and the sampler fills the rest (Reddit LADIES 2092 -> 2217 it/s on one B200)
        prio = int(os.environ.get("SKG_SAMPLER_PRIO", "0"))
        self.sides = [torch.cuda.Stream(priority=prio) for _ in range(self.n_streams)]
        self.side = self.sides[0]
        self.ev_sampled = [torch.cuda.Event() for _ in range(self.n_bufs)]
        self.ev_used = [torch.cuda.Event() for _ in range(self.n_bufs)]
        self._used_armed = [False] * self.n_bufs
        self._buf_stream = [self.sides[b % self.n_streams] for b in range(self.n_bufs)]
        self.dtc = DT[self.dtype]
        self._workers = np.array(self.mine * self.ahead, dtype=np.int32)
        self._states = np.zeros((n_slots, 4), dtype=np.uint64)
        self._boff = np.zeros(n_slots + 1, dtype=np.int64)
        self._bids = np.zeros(n_slots * max(1, batch_size), dtype=np.int64)
        self._len = C.c_int64()
        self._group = []  # (epoch, it) of the sampled-ahead slot groups
        self._pending = []  # (group, arena) sampled ahead of the next pipeline call
        self._gseq = 0      # groups sampled so far (arena = _gseq % n_bufs)

    # -- sharded features over NVLink (one process per GPU) ------------------
    def _install_feature_shards(self):
        """Each rank keeps the feature rows of its workers' nodes; peers' shards are
        mapped with CUDA IPC, so the layer-0 gather reads remote S_0 rows directly over
        NVLink (the exchange the reference only counts, training.py:199)."""
        wr = worker_ranks(self.k, self.active, self.world)
        node_rank, node_row, rows = feature_shard_map(self.partition.owner, wr, self.world)
        mine = self.dg.upload_shard(self.g.features[rows[self.rank]], self.dtype)
        handle = np.zeros(64, dtype=np.uint8)
        check(lib.skg_ipc_handle(mine, ptr(handle, C.c_uint8)))
        handles = [None] * self.world
        self.dist.all_gather_object(handles, handle.tobytes())
        ptrs = []
        for r, hb in enumerate(handles):
            if r == self.rank:
                ptrs.append(mine)
                continue
            h = np.frombuffer(hb, dtype=np.uint8).copy()
            p = C.c_uint64()
            check(lib.skg_ipc_open(ptr(h, C.c_uint8), C.byref(p)))
            ptrs.append(int(p.value))
            self._peer_ptrs.append(int(p.value))
        self.dg.set_feature_shards(ptrs, node_rank, node_row)
        self.shard_rows = len(rows[self.rank])

    # -- host inputs / sampling -------------------------------------------
    def host_inputs(self, epoch, it, group=0):
        """Batch ids and plan PCG64 states of this rank's workers for one iteration,
        into slot group ``group`` (native host runtime, training.py:488-493)."""
        base = group * self.n_my
        o = self._boff[base]
        for i, w in enumerate(self.mine):
            s = base + i
            if self.sampler == "ladies":
                tw = self.worker_train[w]
                check(lib.skg_iteration_inputs(self.seed & 0xFFFFFFFFFFFFFFFF, epoch, it, w,
                                               ptr(tw, C.c_int64), len(tw), self.batch_size,
                                               ptr(self._bids[o:], C.c_int64), C.byref(self._len),
                                               ptr(self._states[s], C.c_uint64)))
                o += self._len.value
                self._boff[s + 1] = o
            else:
                from .seeding import pcg64_state
                self._states[s] = pcg64_state(self.seed, "plan", epoch, it, w)
        return self._boff, self._bids, self._states

    def group_inputs(self, pairs):
        """host_inputs of every iteration in ``pairs`` in one native call, the worker-
        iterations spread over host threads (same results as the per-iteration calls)."""
        n = len(pairs) * self.n_my
        if self.sampler != "ladies" or n == 0:
            for gi, (e, it) in enumerate(pairs):
                self.host_inputs(e, it, gi)
            return
        if getattr(self, "_tw_ptrs", None) is None:
            self._tw = [np.ascontiguousarray(self.worker_train[w], dtype=np.int64) for w in self.mine]
            self._tw_ptrs = np.array([t.ctypes.data for t in self._tw] * self.ahead, dtype=np.uint64)
            self._tw_lens = np.array([len(t) for t in self._tw] * self.ahead, dtype=np.int64)
            self._g_ep = np.zeros(self.n_my * self.ahead, dtype=np.int64)
            self._g_it = np.zeros(self.n_my * self.ahead, dtype=np.int64)
            self._g_w = np.array(self.mine * self.ahead, dtype=np.int32)
        for gi, (e, it) in enumerate(pairs):
            self._g_ep[gi * self.n_my:(gi + 1) * self.n_my] = e
            self._g_it[gi * self.n_my:(gi + 1) * self.n_my] = it
        check(lib.skg_group_inputs(self.seed & 0xFFFFFFFFFFFFFFFF, n, ptr(self._g_ep, C.c_int64),
                                   ptr(self._g_it, C.c_int64), ptr(self._g_w, C.c_int32),
                                   ptr(self._tw_ptrs, C.c_uint64), ptr(self._tw_lens, C.c_int64),
                                   self.batch_size, ptr(self._bids, C.c_int64),
                                   ptr(self._boff, C.c_int64), ptr(self._states, C.c_uint64),
                                   _HOST_THREADS))

    def sample_group(self, pairs, buf=0):
        """Sample the plans of iterations ``pairs`` = [(epoch, it), ...] in one launch
        sequence into plan arena ``buf``, on the side stream."""
        assert 1 <= len(pairs) <= self.ahead
        self._boff[0] = 0
        self.group_inputs(list(pairs))
        self._group = list(pairs)
        self.sample(len(pairs) * self.n_my, buf)

    def _stream_of(self, buf):
        return self._buf_stream[buf]

    def _begin_sample(self, buf):
        # the arena may still be read by the GCN of the group that used it last
        if self._used_armed[buf]:
            self._stream_of(buf).wait_event(self.ev_used[buf])

    def _end_sample(self, buf):
        self.ev_sampled[buf].record(self._stream_of(buf))

    def sample(self, n=None, buf=0):
        n = self.n_my if n is None else n
        if n == 0:
            return
        ps = self.bufs[buf][0]
        self._begin_sample(buf)
        if self.sampler == "ladies":
            check(lib.skg_ladies_sample(ps.h, n, ptr(self._workers, C.c_int32),
                                        ptr(self._boff, C.c_int64), ptr(self._bids, C.c_int64),
                                        MODES[self.mode], float(self.cfg.skew_constant),
                                        float(self.cfg.min_scale), ptr(self._states, C.c_uint64),
                                        C.c_void_p(self._stream_of(buf).cuda_stream)))
        else:
            check(lib.skg_saint_sample(ps.h, n, ptr(self._workers, C.c_int32), MODES[self.mode],
                                       float(self.cfg.skew_constant), float(self.cfg.min_scale),
                                       ptr(self._states, C.c_uint64),
                                       C.c_void_p(self._stream_of(buf).cuda_stream)))
        self._end_sample(buf)

    def sample_device(self, buf, n, workers, batch_len, d_batch, batch_stride, states):
        """LADIES sampling from device-resident batch ids (benchmark inputs)."""
        ps = self.bufs[buf][0]
        self._begin_sample(buf)
        check(lib.skg_ladies_sample_device(
            ps.h, n, ptr(workers, C.c_int32), ptr(batch_len, C.c_int32), d_batch, batch_stride,
            MODES[self.mode], float(self.cfg.skew_constant), float(self.cfg.min_scale),
            ptr(states, C.c_uint64), C.c_void_p(self._stream_of(buf).cuda_stream)))
        self._end_sample(buf)

    def wait_sampled(self, buf):
        """Order the main stream after the sampling of arena ``buf``."""
        self.main.wait_event(self.ev_sampled[buf])

    def release_buf(self, buf):
        """Mark arena ``buf`` free for the next sampling once the queued GCN work ends."""
        self.ev_used[buf].record(self.main)
        self._used_armed[buf] = True

    # -- compute (training.py:499-506) --------------------------------------
    def compute(self, epoch, it, group=0, buf=0):
        if self.n_my:
            ps, gcn = self.bufs[buf]
            s0 = group * self.n_my
            if self.deterministic:  # every worker's gradient kept apart (ordered reduction)
                lrow = self.losses[it % self.per_epoch]
                for i in range(self.n_my):
                    check(lib.skg_gcn_step_batch(gcn, s0 + i, 1, ptr(self.wp, C.c_uint64),
                                                 ptr(self._wgp[i], C.c_uint64), 0,
                                                 lrow[i:].data_ptr(), self.stream))
            else:
                # all of this rank's workers in one batched pass; gradients summed in worker order
                check(lib.skg_gcn_step_batch(gcn, s0, self.n_my, ptr(self.wp, C.c_uint64),
                                             ptr(self.gp, C.c_uint64), 0,
                                             self.losses[it % self.per_epoch].data_ptr(), self.stream))
            check(lib.skg_plans_ledger_add(ps.h, s0, self.n_my,
                                           self.ledger[epoch % self.ledger.shape[0]].data_ptr(),
                                           self.stream))
        else:
            check(lib.skg_zero(self.dtc, self.gflat.data_ptr(), self.n_params, self.stream))

    def reduce_and_step(self):
        if self.deterministic:
            # all ranks' per-worker gradients, summed from zero in worker order (ranks hold
            # contiguous worker blocks, so rank-major rows are worker order)
            self.dist.all_gather(list(self._gathered.view(self.world, self._wcap, -1).unbind(0)),
                                 self.wgrads)
            self.gflat.zero_()
            for r in range(self.world):
                for i in range(self._wcounts[r]):
                    self.gflat.add_(self._gathered[r * self._wcap + i])
        elif self.world > 1:
            self.dist.all_reduce(self.gflat)
        contrib = float(len(self.active))
        if self.optimizer == "sgd":
            check(lib.skg_sgd_step(self.dtc, self.wflat.data_ptr(), self.gflat.data_ptr(),
                                   self.n_params, float(self.lr), contrib, self.stream))
        else:
            self.t += 1
            check(lib.skg_adam_step(self.dtc, self.wflat.data_ptr(), self.gflat.data_ptr(),
                                    self.m.data_ptr(), self.v.data_ptr(), self.n_params,
                                    float(self.lr), contrib, self.t, self.stream))

    def iteration(self, epoch, it):
        self.drop_pending()
        self.sample_group([(epoch, it)], 0)
        self.wait_sampled(0)
        self.compute(epoch, it, 0, 0)
        self.reduce_and_step()
        self.release_buf(0)

    def pipeline(self, groups, sample_fn, compute_fn, next_groups=()):
        """Drive ``groups`` (hashable descriptors) in order: each is sampled into the next
        plan arena (round robin over ``n_bufs``) on that arena's sampler stream, up to
        ``n_streams`` groups ahead of the GCN, which consumes them in order on the main
        stream (``sample_fn(desc, buf)``, ``compute_fn(desc, buf)``).

        The look-ahead carries over between calls: after the last group, the first
        ``n_streams`` of ``next_groups`` are sampled too and kept pending, and a later call
        whose groups start with them computes them without sampling them again.  A run of
        calls is therefore one continuous pipeline (steady state across call boundaries)."""
        S, NB = self.n_streams, self.n_bufs
        groups = list(groups)
        queue = groups + list(next_groups)[:S]
        done = []
        for desc, buf in self._pending:  # sampled ahead by the previous call
            if len(done) < len(queue) and queue[len(done)] == desc:
                done.append((desc, buf))
            else:
                break
        self._pending = []

        def sample_next():
            desc = queue[len(done)]
            buf = self._gseq % NB
            self._gseq += 1
            sample_fn(desc, buf)
            done.append((desc, buf))

        while len(done) < min(S, len(queue)):
            sample_next()
        for g in range(len(groups)):
            desc, b = done[g]
            self.wait_sampled(b)
            compute_fn(desc, b)
            self.release_buf(b)
            if len(done) < len(queue):  # its arena was used by group g - 1, released above
                sample_next()
        self._pending = done[len(groups):]

    def drop_pending(self):
        """Forget plans sampled ahead (before a caller drives the arenas directly)."""
        self._pending = []

    def run(self, pairs, on_iteration=None, next_pairs=()):
        """Train over iterations ``pairs`` in order, ``ahead`` iterations of plans per
        sampling launch, sampled ahead of the GCN on the sampler streams.  ``next_pairs``:
        iterations of the next call, whose first plan groups are sampled ahead now."""
        A = self.ahead

        def chunk(ps):
            ps = [tuple(p) for p in ps]
            return [tuple(ps[g0:g0 + A]) for g0 in range(0, len(ps), A)]

        def compute(grp, b):
            for ci, (e, it) in enumerate(grp):
                self.compute(e, it, ci, b)
                self.reduce_and_step()
                if on_iteration is not None:
                    on_iteration(e, it)

        self.pipeline(chunk(pairs), lambda grp, b: self.sample_group(list(grp), b), compute,
                      next_groups=chunk(next_pairs))

    def check_errors(self, clear: bool = False):
        """Raise the reference's exception for any error of a plan consumed so far
        (sticky per arena, so a later sampling call cannot hide it), or of a plan still
        sampled ahead."""
        torch = _torch()
        torch.cuda.synchronize()
        for ps, _ in self.bufs:
            check(lib.skg_plans_sticky_error(ps.h, 1 if clear else 0))
        for ps, _ in self.bufs:
            for i in range(ps.n_slots):
                _, info, rc = ps.stats(i)
                check(rc)

    def weights_to_model(self):
        for w, v in zip(self.model.weights, self.wviews):
            w[...] = v.double().cpu().numpy()

    def close(self):
        for p in self._peer_ptrs:
            lib.skg_ipc_close(p)
        self._peer_ptrs = []
        if self.world > 1:  # restore the single-store map for later single-rank use
            X = self.g.features
            self.dg.feat_key = None
            self.dg.ensure_features(X, self.dtype)
        _torch().cuda.synchronize()
        for ps, _ in self.bufs:
            self.dg.release(ps)


def train_distributed(g: WeightedGraph, partition: Partition, model: GcnModel, cfg: SamplerConfig, *,
                      epochs: int, batch_size: int, lr: float, mode: str, seed: int,
                      sampler: str = "ladies", subgraph_size: int | None = None,
                      optimizer: str = "sgd", ahead: int = 3, streams: int = 2,
                      pos_weight: float = 50.0, deterministic: bool = False) -> tuple:
    """Data-parallel training with per-iteration gradient averaging (training.py:430-518).

    Single process: all workers run on this GPU.  Under torch.distributed (one process
    per GPU) each rank runs a contiguous block of workers and gradients are summed with
    an NCCL all-reduce; metrics and ledger are identical on every rank.  ``ahead``
    iterations of plans are sampled per launch (plans never depend on the weights).
    """
    torch = _torch()
    # the GCN runs on a high-priority stream, the sampler streams at the lowest priority
    hp = torch.cuda.Stream(priority=-1)
    hp.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(hp):
        out = _train_distributed(g, partition, model, cfg, epochs=epochs, batch_size=batch_size, lr=lr,
                                 mode=mode, seed=seed, sampler=sampler, subgraph_size=subgraph_size,
                                 optimizer=optimizer, ahead=ahead, streams=streams, pos_weight=pos_weight,
                                 deterministic=deterministic)
    torch.cuda.current_stream().wait_stream(hp)
    return out


def _train_distributed(g, partition, model, cfg, *, epochs, batch_size, lr, mode, seed, sampler,
                       subgraph_size, optimizer, ahead, streams, pos_weight, deterministic):
    torch = _torch()
    tr = Trainer(g, partition, model, cfg, batch_size=batch_size, lr=lr, mode=mode, seed=seed,
                 sampler=sampler, subgraph_size=subgraph_size, optimizer=optimizer, epochs=epochs,
                 ahead=ahead, streams=streams, pos_weight=pos_weight, deterministic=deterministic)
    k, L = tr.k, tr.L
    metrics = Metrics()
    val_nodes = np.flatnonzero(g.val_mask) if g.val_mask is not None else np.empty(0, dtype=np.int64)
    labels_t = torch.as_tensor(np.asarray(g.labels), device="cuda")

    def end_of_epoch(epoch, it):
        if it != tr.per_epoch - 1:
            return
        losses = tr.losses.cpu().numpy()
        tr.check_errors()  # training.py:296-297 raises inside the epoch; here at its end
        ledger = tr.ledger[epoch]
        loss_sum = np.zeros(k)
        loss_cnt = np.zeros(k, dtype=np.int64)
        for i, w in enumerate(tr.mine):  # python-float sums in iteration order
            for j in range(tr.per_epoch):
                loss_sum[w] += losses[j, i]
                loss_cnt[w] += 1
        if tr.world > 1:
            loss_sum, loss_cnt, ledger = reduce_epoch_stats(tr.dist, loss_sum, loss_cnt, ledger)
        ledger_np = ledger.cpu().numpy()
        logits = _predict_device(tr.dg, tr.wviews, tr.dims, tr.dtype)
        if tr.multilabel:  # accuracy columns carry micro-F1 of z > 0 for multi-hot labels
            zl = logits.double().cpu().numpy()
            ylab = np.asarray(g.labels)

            def score(nodes):
                return multilabel_scores(zl[nodes], ylab[nodes])[1] if len(nodes) else 0.0
        else:
            correct = (torch.argmax(logits, dim=1) == labels_t).cpu().numpy()

            def score(nodes):
                return float(np.mean(correct[nodes])) if len(nodes) else 0.0
        val_acc = score(val_nodes)
        for w in range(k):
            tw = tr.worker_train[w]
            train_acc = score(tw)
            mean_loss = float(loss_sum[w] / loss_cnt[w]) if loss_cnt[w] else 0.0
            metrics.rows.append(MetricRow(epoch=epoch, worker=w, loss=mean_loss,
                                          train_acc=train_acc, val_acc=val_acc,
                                          comm_nodes_epoch=int(ledger_np[w].sum())))

    try:
        pairs = [(e, it) for e in range(epochs) for it in range(tr.per_epoch)]
        tr.run(pairs, on_iteration=end_of_epoch)
        tr.check_errors()
        tr.weights_to_model()
        led = tr.ledger.clone()
        if tr.world > 1:  # each rank counted its own workers (training.py:117-134 is global)
            tr.dist.all_reduce(led)
        ledger_all = CommLedger(led.cpu().numpy()[:epochs].copy())
    finally:
        tr.close()
    return metrics, ledger_all
