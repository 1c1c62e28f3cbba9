"""Generate golden vectors from the UNMODIFIED reference (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (``/root/reference/pkg/src/skewgcn``) is importable only here, not on
the GPU box, so its outputs are frozen into ``tests/golden/*.npz``.  Inputs are
either stored verbatim (small edge lists) or regenerated deterministically from
``paper_2101_07706_b200.synth`` (large shaped graphs; the structure hash is
recorded and re-checked by the tests).  Plans are driven by numpy generators
whose construction is recorded (``default_rng(seed)`` or ``spawn_rng`` labels).

Floating outputs that go through BLAS (losses, gradients, weights) are stored as
values and compared at a tolerance; integer/index outputs and the sampler's
IEEE-only float arithmetic (q, block values) are compared exactly.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
import warnings
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

import skewgcn as sg  # noqa: E402  (reference, read-only)

from paper_2101_07706_b200.synth import make_shaped_graph  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_graph_from_edges(edges, n):
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "edges.txt"
        p.write_text("".join(f"{u} {v}\n" for u, v in edges), encoding="utf-8")
        g = sg.load_edge_list(p, n_hint=n)
    return sg.normalize_weights(g)


def er_edges(n, p, seed):
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, k=1)
    keep = rng.random(len(iu)) < p
    return np.stack([iu[keep], ju[keep]], axis=1).astype(np.int64)


def ref_graph_from_shaped(sgph):
    feats = sgph.features.astype(np.float64) if sgph.features.shape[1] else None
    labels = sgph.labels if np.ndim(sgph.labels) == 1 else None  # multi-hot: no reference head
    return sg.WeightedGraph(n_nodes=sgph.n_nodes, offsets=sgph.offsets,
                            neighbors=sgph.neighbors.astype(np.int64),
                            weights=sgph.weights, normalized=True,
                            features=feats,
                            labels=labels, train_mask=sgph.train_mask,
                            val_mask=sgph.val_mask, test_mask=sgph.test_mask)


def make_rng(spec):
    """("default", seed) | ("spawn", seed, *labels) | ("philox", key, skip) |
    ("mt19937", seed) | ("sfc64", seed); `skip` next_uint64 outputs are consumed first so
    the Philox buffer is part-used (buffer_pos != 4)."""
    if spec[0] == "default":
        return np.random.default_rng(spec[1])
    if spec[0] == "philox":
        g = np.random.Generator(np.random.Philox(key=spec[1]))
        g.bit_generator.random_raw(spec[2])
        return g
    if spec[0] == "mt19937":
        return np.random.Generator(np.random.MT19937(spec[1]))
    if spec[0] == "sfc64":
        return np.random.Generator(np.random.SFC64(spec[1]))
    return sg.spawn_rng(spec[1], *spec[2:])


class Store:
    def __init__(self):
        self.arrays = {}
        self.meta = {}

    def put(self, case, key, arr):
        self.arrays[f"{case}/{key}"] = np.asarray(arr)

    def save(self, path):
        self.arrays["__meta__"] = np.array(json.dumps(self.meta))
        np.savez_compressed(path, **self.arrays)
        print("wrote", path, os.path.getsize(path), "bytes", len(self.meta), "cases")


def dump_plan(st, case, plan, full_dist=True):
    st.put(case, "batch", plan.batch)
    st.put(case, "starvation", np.int64(plan.starvation_events))
    st.put(case, "remote", plan.remote_per_layer())
    for l, L in enumerate(plan.layers):
        b = L.block.tocsr()
        st.put(case, f"L{l}/nodes", L.nodes)
        st.put(case, f"L{l}/indptr", b.indptr.astype(np.int64))
        st.put(case, f"L{l}/indices", b.indices.astype(np.int64))
        st.put(case, f"L{l}/data", b.data)
        st.put(case, f"L{l}/shape", np.array(b.shape, dtype=np.int64))
        has = L.dist is not None
        st.put(case, f"L{l}/has_dist", np.int64(has))
        if has:
            st.put(case, f"L{l}/n_cand", np.int64(len(L.dist.candidates)))
            st.put(case, f"L{l}/q_sha", np.array(sha(L.dist.q)))
            st.put(case, f"L{l}/cand_sha", np.array(sha(L.dist.candidates)))
            st.put(case, f"L{l}/s_used", np.float64(L.dist.s_used))
            if full_dist:
                st.put(case, f"L{l}/q", L.dist.q)
                st.put(case, f"L{l}/cand", L.dist.candidates)


# ---------------------------------------------------------------------------


def small_cases(st: Store):
    """ER / SBM graphs: every mode, saturated and sampled layers, edge cases."""
    graphs = {
        "er20": (20, er_edges(20, 0.25, 0)),
        "er30": (30, er_edges(30, 0.25, 3)),
        "er60": (60, er_edges(60, 0.10, 11)),
        "er200": (200, er_edges(200, 0.05, 5)),
        "path3": (3, np.array([[0, 1], [1, 2]])),
        "iso6": (6, np.zeros((0, 2), dtype=np.int64)),
    }
    for gname, (n, e) in graphs.items():
        st.put("graph_" + gname, "edges", e)
        st.put("graph_" + gname, "n", np.int64(n))
    idx = 0
    combos = [
        # graph, k, strategy, pseed, worker, batch spec, budget, mode, D, min_scale, layers, rng
        ("er20", 2, "contiguous", None, 0, ("owned", 4), 21, "full", 0.0, 1.0, 2, ("default", 0)),
        ("er20", 1, "contiguous", None, 0, ("arange", 4), 6, "full", 0.0, 1.0, 2, ("default", 3)),
        ("er20", 1, "contiguous", None, 0, ("arange", 4), 6, "skewed", 8.0, 1.0, 2, ("default", 3)),
        ("er30", 3, "random", 4, 1, ("owned", 4), 5, "local", 0.0, 1.0, 3, ("default", 2)),
        ("er30", 3, "random", 4, 1, ("owned", 4), 5, "skewed", 4.0, 1.0, 3, ("default", 7)),
        ("er60", 4, "random", 31, 0, ("owned", 12), 16, "skewed", 8.0, 1.0, 3, ("default", 1000)),
        ("er60", 4, "random", 31, 0, ("owned", 12), 16, "full", 0.0, 1.0, 3, ("default", 1001)),
        ("er60", 2, "hash", None, 1, ("owned", 9), 7, "local", 0.0, 1.0, 4, ("default", 5)),
        ("er200", 4, "random", 9, 2, ("owned", 40), 32, "skewed", 16.0, 1.0, 5, ("spawn", 0, "plan", 0, 1, 2)),
        ("er200", 4, "random", 9, 2, ("owned", 40), 32, "skewed", 0.0, 1.0, 5, ("spawn", 0, "plan", 0, 1, 2)),
        ("er200", 4, "random", 9, 2, ("owned", 40), 32, "skewed", 2.0, 3.5, 5, ("spawn", 0, "plan", 0, 1, 2)),
        ("er200", 4, "random", 9, 3, ("owned", 40), 32, "local", 0.0, 1.0, 5, ("default", 77)),
        ("er200", 8, "hash", None, 5, ("owned", 25), 3, "full", 0.0, 1.0, 5, ("default", 78)),
        ("er200", 2, "random", 1, 0, ("owned", 100), 1, "skewed", 8.0, 1.0, 3, ("default", 79)),
        ("path3", 1, "contiguous", None, 0, ("arange", 1), 2, "full", 0.0, 1.0, 2, ("default", 0)),
        ("iso6", 2, "contiguous", None, 0, ("arange", 6), 10, "full", 0.0, 1.0, 1, ("default", 0)),
        ("iso6", 2, "contiguous", None, 1, ("arange", 6), 2, "local", 0.0, 1.0, 2, ("default", 0)),
    ]
    for (gname, k, strat, pseed, worker, bspec, budget, mode, D, ms, nl, rspec) in combos:
        n, e = graphs[gname]
        g = ref_graph_from_edges([tuple(x) for x in e.tolist()], n)
        part = sg.partition_nodes(n, k, strat, seed=pseed)
        batch = part.owned_by(worker)[: bspec[1]] if bspec[0] == "owned" else np.arange(bspec[1])
        cfg = sg.SamplerConfig(budget=budget, mode=mode, skew_constant=D, min_scale=ms)
        plan = sg.ladies_plan(g, part, worker, batch, cfg, nl, make_rng(rspec))
        case = f"ladies_{idx:02d}"
        st.meta[case] = dict(kind="ladies", graph=gname, k=k, strategy=strat, pseed=pseed,
                             worker=worker, batch=batch.tolist(), budget=budget, mode=mode,
                             D=D, min_scale=ms, n_layers=nl, rng=list(rspec))
        dump_plan(st, case, plan)
        idx += 1

    # local starvation with a worker owning nothing (test_training.py:92-102)
    g = ref_graph_from_edges([(0, 1)], 2)
    st.put("graph_k2", "edges", np.array([[0, 1]]))
    st.put("graph_k2", "n", np.int64(2))
    part = sg.Partition(n_workers=2, owner=np.array([1, 1]))
    plan = sg.ladies_plan(g, part, 0, np.array([1]), sg.SamplerConfig(budget=2, mode="local"), 2,
                          np.random.default_rng(0))
    st.meta["ladies_starve"] = dict(kind="ladies", graph="k2", k=2, strategy="explicit",
                                    owner=[1, 1], worker=0, batch=[1], budget=2, mode="local",
                                    D=0.0, min_scale=1.0, n_layers=2, rng=["default", 0])
    dump_plan(st, "ladies_starve", plan)

    # SAINT plans (training.py:216-254)
    idx = 0
    for (gname, k, strat, pseed, worker, size, budget, mode, D, nl, rspec, pre) in [
        ("er60", 2, "random", 1, 0, 10, 8, "full", 0.0, 2, ("default", 2), False),
        ("er60", 2, "random", 1, 0, 10, 8, "skewed", 0.0, 2, ("default", 2), False),
        ("er60", 2, "random", 3, 1, 15, 8, "skewed", 8.0, 3, ("default", 9), True),
        ("er200", 4, "random", 5, 2, 50, 8, "local", 0.0, 2, ("default", 6), False),
        ("er200", 4, "random", 5, 3, 300, 8, "full", 0.0, 2, ("default", 6), False),
        ("er200", 4, "hash", None, 0, 60, 8, "skewed", 4.0, 3, ("spawn", 0, "plan", 1, 2, 0), True),
    ]:
        n, e = graphs[gname]
        g = ref_graph_from_edges([tuple(x) for x in e.tolist()], n)
        part = sg.partition_nodes(n, k, strat, seed=pseed)
        train = np.arange(n) if gname != "er200" else np.arange(0, n, 2)
        cfg = sg.SamplerConfig(budget=budget, mode=mode, skew_constant=D)
        norms = sg.training.train_column_norms(g, train) if pre else None
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            plan = sg.saint_plan(g, part, worker, train, size, cfg, nl, make_rng(rspec),
                                 norms=norms)
        case = f"saint_{idx:02d}"
        st.meta[case] = dict(kind="saint", graph=gname, k=k, strategy=strat, pseed=pseed,
                             worker=worker, train=train.tolist(), size=size, budget=budget,
                             mode=mode, D=D, min_scale=1.0, n_layers=nl, rng=list(rspec),
                             precomputed=pre)
        dump_plan(st, case, plan)
        idx += 1

    # forward / loss_and_backward (training.py:261-318)
    for i, (gname, k, mode, budget, dims, mseed, rseed) in enumerate([
        ("er20", 2, "full", 6, [4, 5, 5, 3], 9, 8),
        ("er20", 3, "skewed", 6, [4, 5, 5, 3], 9, 8),
        ("er60", 2, "local", 7, [6, 8, 4], 1, 3),
        ("er200", 4, "skewed", 32, [16, 12, 12, 12, 12, 5], 2, 4),
    ]):
        n, e = graphs[gname]
        g = ref_graph_from_edges([tuple(x) for x in e.tolist()], n)
        rng = np.random.default_rng(100 + i)
        g.features = rng.normal(size=(n, dims[0]))
        g.labels = rng.integers(0, dims[-1], size=n)
        g.labels[rng.random(n) < 0.2] = -1
        part = sg.partition_nodes(n, k, "random", seed=7)
        batch = part.owned_by(0)[: max(4, n // 10)]
        if not np.any(g.labels[batch] >= 0):
            g.labels[batch[0]] = 0
        cfg = sg.SamplerConfig(budget=budget, mode=mode, skew_constant=4.0)
        plan = sg.ladies_plan(g, part, 0, batch, cfg, len(dims) - 1, np.random.default_rng(rseed))
        model = sg.init_model(dims, seed=mseed)
        loss, grads = sg.loss_and_backward(model, plan, g.features, g.labels)
        logits = sg.forward(model, plan, g.features)
        case = f"fb_{i:02d}"
        st.meta[case] = dict(kind="fb", graph=gname, k=k, strategy="random", pseed=7, worker=0,
                             batch=batch.tolist(), budget=budget, mode=mode, D=4.0,
                             min_scale=1.0, n_layers=len(dims) - 1, rng=["default", rseed],
                             dims=dims, model_seed=mseed, data_seed=100 + i)
        dump_plan(st, case, plan)
        st.put(case, "features", g.features)
        st.put(case, "labels", g.labels)
        st.put(case, "loss", np.float64(loss))
        st.put(case, "logits", logits)
        for l, gr in enumerate(grads):
            st.put(case, f"grad{l}", gr)

    # simulated distributed training (training.py:430-518) on reference SBMs
    for i, (n, blocks, k, mode, sampler, opt, epochs, bs, lr, D, budget, sub) in enumerate([
        (80, 2, 2, "skewed", "ladies", "sgd", 3, 8, 0.2, 4.0, 8, None),
        (100, 2, 4, "full", "ladies", "sgd", 2, 10, 0.5, 0.0, 12, None),
        (100, 2, 4, "local", "ladies", "sgd", 2, 10, 0.1, 0.0, 8, None),
        (80, 2, 2, "full", "ladies", "adam", 2, 8, 0.01, 0.0, 8, None),
        (120, 3, 3, "skewed", "saint", "sgd", 2, 8, 0.3, 8.0, 8, 20),
    ]):
        spec = sg.SbmSpec(n_nodes=n, n_blocks=blocks, p_in=0.2, p_out=0.02, feature_dim=8,
                          noise_sigma=0.3, seed=i)
        g = sg.synth_sbm(spec)
        part = sg.partition_nodes(n, k, "random", seed=1 + i)
        model = sg.init_model([g.feature_dim, 8, 6, blocks], seed=5 + i)
        cfg = sg.SamplerConfig(budget=budget, mode=mode, skew_constant=D)
        metrics, ledger = sg.train_distributed(g, part, model, cfg, epochs=epochs, batch_size=bs,
                                               lr=lr, mode=mode, seed=11 + i, sampler=sampler,
                                               subgraph_size=sub, optimizer=opt)
        case = f"train_{i:02d}"
        st.meta[case] = dict(kind="train", n=n, blocks=blocks, k=k, pseed=1 + i, mode=mode,
                             sampler=sampler, optimizer=opt, epochs=epochs, batch_size=bs, lr=lr,
                             D=D, budget=budget, subgraph_size=sub, dims=[8, 8, 6, blocks],
                             model_seed=5 + i, seed=11 + i)
        st.put(case, "offsets", g.offsets)
        st.put(case, "neighbors", g.neighbors)
        st.put(case, "weights", g.weights)
        st.put(case, "features", g.features)
        st.put(case, "labels", g.labels)
        st.put(case, "train_mask", g.train_mask)
        st.put(case, "val_mask", g.val_mask)
        st.put(case, "ledger", ledger.counts)
        st.put(case, "metrics", np.array([[r.epoch, r.worker, r.loss, r.train_acc, r.val_acc,
                                            r.comm_nodes_epoch] for r in metrics.rows]))
        for l, w in enumerate(model.weights):
            st.put(case, f"w{l}", w)


def shaped_cases(st: Store, shapes):
    """Benchmark-shaped graphs from the O(m) generator, reference plans on top."""
    for shape, k, runs, sampler in shapes:
        # plans never read features; the large shapes skip them (YouTube's would be 18 GB)
        sgph = make_shaped_graph(shape, seed=0, with_features=shape not in ("youtube", "amazon"))
        g = ref_graph_from_shaped(sgph)
        case_g = f"shape_{shape}"
        st.meta[case_g] = dict(kind="shape", shape=shape, seed=0,
                               structure_sha=sgph.structure_hash(), nnz=sgph.nnz,
                               weights_sha=sha(sgph.weights))
        part = sg.partition_nodes(sgph.n_nodes, k, "random", seed=1)
        st.meta[case_g]["owner_sha"] = sha(part.owner)
        if shape == "cora":  # the generator's normalisation equals the reference's
            und = sg.undirected_edges(sg.WeightedGraph(
                n_nodes=sgph.n_nodes, offsets=sgph.offsets, neighbors=sgph.neighbors,
                weights=sgph.weights))
            und = und[und[:, 0] != und[:, 1]]
            g2 = ref_graph_from_edges([tuple(x) for x in und.tolist()], sgph.n_nodes)
            assert np.array_equal(g2.offsets, g.offsets)
            assert np.array_equal(g2.neighbors, g.neighbors)
            assert np.array_equal(g2.weights, g.weights)
        all_train = np.flatnonzero(g.train_mask)
        saint_norms = None
        for j, (mode, D, epoch, it, worker) in enumerate(runs):
            cfg = sg.SamplerConfig(budget=512 if sampler == "ladies" else 4500,
                                   mode=mode, skew_constant=D)
            if sampler == "ladies":
                wt = np.flatnonzero(g.train_mask & (part.owner == worker))
                take = min(512, len(wt))
                batch = sg.node_set(sg.spawn_rng(0, "batch", epoch, it, worker).choice(
                    wt, size=take, replace=False))
                plan = sg.ladies_plan(g, part, worker, batch, cfg, 5,
                                      sg.spawn_rng(0, "plan", epoch, it, worker))
            else:
                if saint_norms is None and mode != "local":
                    saint_norms = sg.training.train_column_norms(g, all_train)
                    st.put(case_g, "saint_norms_sha", np.array(sha(saint_norms)))
                plan = sg.saint_plan(g, part, worker, all_train, 4500, cfg, 5,
                                     sg.spawn_rng(0, "plan", epoch, it, worker),
                                     norms=None if mode == "local" else saint_norms)
            case = f"{shape}_{sampler}_{j:02d}"
            st.meta[case] = dict(kind=f"shaped_{sampler}", shape=shape, k=k, pseed=1, mode=mode,
                                 D=D, epoch=epoch, it=it, worker=worker, seed=0,
                                 budget=cfg.budget, n_layers=5)
            dump_plan(st, case, plan, full_dist=(shape == "cora"))
            print(case, [len(L.nodes) for L in plan.layers], plan.remote_per_layer().tolist(),
                  flush=True)


def rng_cases(st: Store):
    """Plans driven by non-PCG64 Generators (the reference accepts any numpy Generator,
    training.py:162-164, 216-219): Philox (fresh and with a part-used output buffer),
    MT19937 and SFC64.  `after` = the next 4 random() values of the generator after the
    plan, which pins how far the plan advanced it."""
    n, e = 200, er_edges(200, 0.05, 5)
    st.put("graph_er200", "edges", e)
    st.put("graph_er200", "n", np.int64(n))
    g = ref_graph_from_edges([tuple(x) for x in e.tolist()], n)
    idx = 0
    for kind, mode, D, rspec in [
        ("ladies", "skewed", 8.0, ("philox", 12345, 0)),
        ("ladies", "skewed", 8.0, ("philox", 7, 3)),
        ("ladies", "full", 0.0, ("philox", 2**64 - 1, 1)),
        ("ladies", "skewed", 4.0, ("mt19937", 3)),
        ("ladies", "local", 0.0, ("sfc64", 9)),
        ("saint", "skewed", 8.0, ("philox", 99, 2)),
        ("saint", "full", 0.0, ("mt19937", 5)),
    ]:
        part = sg.partition_nodes(n, 4, "random", seed=9)
        rng = make_rng(rspec)
        if kind == "ladies":
            batch = part.owned_by(2)[:40]
            cfg = sg.SamplerConfig(budget=32, mode=mode, skew_constant=D)
            plan = sg.ladies_plan(g, part, 2, batch, cfg, 5, rng)
            meta = dict(kind="ladies", graph="er200", k=4, strategy="random", pseed=9, worker=2,
                        batch=batch.tolist(), budget=32, mode=mode, D=D, min_scale=1.0,
                        n_layers=5, rng=list(rspec))
        else:
            train = np.arange(0, n, 2)
            cfg = sg.SamplerConfig(budget=8, mode=mode, skew_constant=D)
            plan = sg.saint_plan(g, part, 1, train, 30, cfg, 3, rng)
            meta = dict(kind="saint", graph="er200", k=4, strategy="random", pseed=9, worker=1,
                        train=train.tolist(), size=30, budget=8, mode=mode, D=D, min_scale=1.0,
                        n_layers=3, rng=list(rspec), precomputed=False)
        case = f"rng_{idx:02d}"
        st.meta[case] = meta
        dump_plan(st, case, plan)
        st.put(case, "after", rng.random(4))
        idx += 1


def reddit_fb_cases(st: Store):
    """loss_and_backward / forward (training.py:261-318) at the benchmarked configuration:
    Reddit-shaped graph, dims [602, 256, 256, 256, 256, 41], init_model seed 0, the synth
    features, on the golden_reddit plans (skewed D=8 / full / local).  Gradients are
    stored in full for the skewed plan (the bench's mode); for every plan a seeded sample
    of 8192 entries per layer plus each layer's Frobenius norm."""
    sgph = make_shaped_graph("reddit", seed=0)
    g = ref_graph_from_shaped(sgph)
    part = sg.partition_nodes(sgph.n_nodes, 8, "random", seed=1)
    dims = [602, 256, 256, 256, 256, 41]
    model = sg.init_model(dims, seed=0)
    st.meta["shape_reddit"] = dict(kind="shape", shape="reddit", seed=0,
                                   structure_sha=sgph.structure_hash(),
                                   features_sha=sgph.features_hash())
    for j, (mode, D, worker) in enumerate([("skewed", 8.0, 0), ("full", 0.0, 1), ("local", 0.0, 2)]):
        cfg = sg.SamplerConfig(budget=512, mode=mode, skew_constant=D)
        wt = np.flatnonzero(g.train_mask & (part.owner == worker))
        batch = sg.node_set(sg.spawn_rng(0, "batch", 0, 0, worker).choice(
            wt, size=min(512, len(wt)), replace=False))
        plan = sg.ladies_plan(g, part, worker, batch, cfg, 5, sg.spawn_rng(0, "plan", 0, 0, worker))
        loss, grads = sg.loss_and_backward(model, plan, g.features, g.labels)
        logits = sg.forward(model, plan, g.features)
        case = f"reddit_fb_{j:02d}"
        st.meta[case] = dict(kind="reddit_fb", mode=mode, D=D, worker=worker, epoch=0, it=0,
                             seed=0, k=8, pseed=1, budget=512, n_layers=5, dims=dims,
                             model_seed=0, full_grads=j == 0)
        st.put(case, "batch", plan.batch)
        st.put(case, "remote", plan.remote_per_layer())
        st.put(case, "loss", np.float64(loss))
        st.put(case, "logits", logits)
        sel = np.random.default_rng(1234)
        for l, gr in enumerate(grads):
            idx = sel.choice(gr.size, size=min(8192, gr.size), replace=False)
            st.put(case, f"grad{l}_idx", idx.astype(np.int64))
            st.put(case, f"grad{l}_val", gr.reshape(-1)[idx])
            st.put(case, f"grad{l}_norm", np.float64(np.linalg.norm(gr)))
            if j == 0:
                st.put(case, f"grad{l}", gr)
        print(case, loss, flush=True)


def reddit_pipeline_cases(st: Store, iters=3, k=8):
    """Every worker's plan of iterations (0, 0..iters-1) at the Reddit shape, k = 8,
    skewed D = 8 (the bench's 24-plan look-ahead group), and the ledger they make
    (training.py:486-499): the CUDA Trainer pipeline must reproduce them bit for bit."""
    sgph = make_shaped_graph("reddit", seed=0, with_features=False)
    g = sg.WeightedGraph(n_nodes=sgph.n_nodes, offsets=sgph.offsets,
                         neighbors=sgph.neighbors.astype(np.int64), weights=sgph.weights,
                         normalized=True, train_mask=sgph.train_mask)
    part = sg.partition_nodes(sgph.n_nodes, k, "random", seed=1)
    cfg = sg.SamplerConfig(budget=512, mode="skewed", skew_constant=8.0)
    ledger = np.zeros((k, 5), dtype=np.int64)
    st.meta["pipeline"] = dict(kind="pipeline", shape="reddit", k=k, pseed=1, mode="skewed",
                               D=8.0, budget=512, batch_size=512, n_layers=5, seed=0,
                               iters=iters, structure_sha=sgph.structure_hash())
    for it in range(iters):
        for w in range(k):
            wt = np.flatnonzero(g.train_mask & (part.owner == w))
            batch = sg.node_set(sg.spawn_rng(0, "batch", 0, it, w).choice(
                wt, size=min(512, len(wt)), replace=False))
            plan = sg.ladies_plan(g, part, w, batch, cfg, 5, sg.spawn_rng(0, "plan", 0, it, w))
            ledger[w] += plan.remote_per_layer()
            case = f"pipe_{it}_{w}"
            st.put(case, "batch", plan.batch.astype(np.int32))
            st.put(case, "remote", plan.remote_per_layer())
            for l, L in enumerate(plan.layers):
                b = L.block.tocsr()
                st.put(case, f"L{l}/nodes", L.nodes.astype(np.int32))
                st.put(case, f"L{l}/indptr", b.indptr.astype(np.int32))
                st.put(case, f"L{l}/indices", b.indices.astype(np.int32))
                st.put(case, f"L{l}/data", b.data)
                st.put(case, f"L{l}/q_sha", np.array(sha(L.dist.q) if L.dist is not None else ""))
            print(case, [len(L.nodes) for L in plan.layers], flush=True)
    st.put("pipeline", "ledger", ledger)


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "cora", "reddit_s", "amazon_s", "reddit"]
    if "reddit_fb" in which:
        st = Store()
        reddit_fb_cases(st)
        st.save(HERE / "golden_reddit_fb.npz")
    if "pipeline" in which:
        st = Store()
        reddit_pipeline_cases(st)
        st.save(HERE / "golden_pipeline.npz")
    if "rng" in which:
        st = Store()
        rng_cases(st)
        st.save(HERE / "golden_rng.npz")
    if "small" in which:
        st = Store()
        small_cases(st)
        st.meta["__versions__"] = dict(numpy=np.__version__, scipy=__import__("scipy").__version__)
        st.save(HERE / "golden_small.npz")
    for shape, k, runs, sampler in [
        ("cora", 4, [("full", 0.0, 0, 0, 0), ("skewed", 4.0, 0, 0, 0), ("local", 0.0, 0, 0, 1),
                     ("skewed", 4.0, 1, 3, 2), ("full", 0.0, 2, 1, 3)], "ladies"),
        ("reddit_s", 8, [("full", 0.0, 0, 0, 0), ("skewed", 8.0, 0, 0, 0), ("local", 0.0, 0, 1, 3),
                         ("skewed", 32.0, 0, 2, 7)], "ladies"),
        ("amazon_s", 8, [("full", 0.0, 0, 0, 0), ("skewed", 8.0, 0, 0, 1), ("local", 0.0, 0, 1, 2)],
         "saint"),
        ("reddit", 8, [("skewed", 8.0, 0, 0, 0), ("full", 0.0, 0, 0, 1), ("local", 0.0, 0, 0, 2)],
         "ladies"),
        # > 16 x 65536 nodes: the device takes the global-atomic expand path
        ("youtube", 8, [("skewed", 8.0, 0, 0, 0), ("full", 0.0, 0, 1, 3), ("local", 0.0, 0, 2, 5)],
         "ladies"),
        # the full Amazon shape (1.6M nodes, 132M CSR entries), GraphSAINT subgraph 4500
        ("amazon", 8, [("skewed", 8.0, 0, 0, 1)], "saint"),
    ]:
        if shape in which:
            st = Store()
            shaped_cases(st, [(shape, k, runs, sampler)])
            st.save(HERE / f"golden_{shape}.npz")
