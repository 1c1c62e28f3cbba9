"""Pin the CPU oracle against golden vectors produced by the unmodified reference."""

import warnings

import numpy as np
import pytest

import skewgcn_oracle as O
from golden_util import (assert_plan_equal, cfg_for, golden, make_rng, oracle_graph_from_shaped,
                         partition_for, plan_to_dict, shaped, shaped_batch, small_graph)

G = golden("small")


@pytest.mark.parametrize("case", G.cases("ladies"))
def test_ladies_small(case):
    m = G.meta[case]
    g = small_graph(m["graph"])
    part = partition_for(m, g.n_nodes)
    plan = O.ladies_plan(g, part, m["worker"], np.array(m["batch"], dtype=np.int64), cfg_for(m),
                         m["n_layers"], make_rng(m["rng"]))
    assert_plan_equal(plan_to_dict(plan), G.expected_plan(case))


@pytest.mark.parametrize("case", G.cases("saint"))
def test_saint_small(case):
    m = G.meta[case]
    g = small_graph(m["graph"])
    part = partition_for(m, g.n_nodes)
    train = np.array(m["train"], dtype=np.int64)
    norms = O.column_norms(g, train, train) if m["precomputed"] else None
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        plan = O.saint_plan(g, part, m["worker"], train, m["size"], cfg_for(m), m["n_layers"],
                            make_rng(m["rng"]), norms=norms)
    assert_plan_equal(plan_to_dict(plan), G.expected_plan(case))


@pytest.mark.parametrize("case", G.cases("fb"))
def test_forward_backward_small(case):
    m = G.meta[case]
    g = small_graph(m["graph"])
    part = partition_for(m, g.n_nodes)
    plan = O.ladies_plan(g, part, m["worker"], np.array(m["batch"], dtype=np.int64), cfg_for(m),
                         m["n_layers"], make_rng(m["rng"]))
    assert_plan_equal(plan_to_dict(plan), G.expected_plan(case))
    x = G.get(case, "features")
    y = G.get(case, "labels")
    ws = O.init_model(m["dims"], m["model_seed"])
    loss, grads = O.loss_and_backward(ws, plan, x, y)
    np.testing.assert_allclose(O.forward(ws, plan, x), G.get(case, "logits"), rtol=1e-12,
                               atol=1e-14)
    assert loss == pytest.approx(float(G.get(case, "loss")), rel=1e-12)
    for l, gr in enumerate(grads):
        np.testing.assert_allclose(gr, G.get(case, f"grad{l}"), rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("case", G.cases("train"))
def test_train_distributed_small(case):
    m = G.meta[case]
    g = O.Graph(n_nodes=m["n"], offsets=G.get(case, "offsets"), neighbors=G.get(case, "neighbors"),
                weights=G.get(case, "weights"), normalized=True, features=G.get(case, "features"),
                labels=G.get(case, "labels"), train_mask=G.get(case, "train_mask"),
                val_mask=G.get(case, "val_mask"))
    part = O.partition_nodes(m["n"], m["k"], "random", seed=m["pseed"])
    ws = O.init_model(m["dims"], m["model_seed"])
    cfg = O.SamplerConfig(budget=m["budget"], skew_constant=m["D"], mode=m["mode"])
    rows, ledger = O.train_distributed(g, part, ws, cfg, epochs=m["epochs"],
                                       batch_size=m["batch_size"], lr=m["lr"], mode=m["mode"],
                                       seed=m["seed"], sampler=m["sampler"],
                                       subgraph_size=m["subgraph_size"], optimizer=m["optimizer"])
    np.testing.assert_array_equal(ledger, G.get(case, "ledger"))
    got = np.array([[r.epoch, r.worker, r.loss, r.train_acc, r.val_acc, r.comm_nodes_epoch]
                    for r in rows])
    np.testing.assert_allclose(got, G.get(case, "metrics"), rtol=1e-9, atol=1e-12)
    for l, w in enumerate(ws):
        np.testing.assert_allclose(w, G.get(case, f"w{l}"), rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("shape", ["cora", "reddit_s", "amazon_s", "youtube", "amazon"])
def test_shaped_plans(shape):
    G2 = golden(shape)
    gm = G2.meta[f"shape_{shape}"]
    sgph = shaped(shape)
    assert sgph.structure_hash() == gm["structure_sha"], "generator drifted from the golden graph"
    g = oracle_graph_from_shaped(sgph)
    cases = G2.cases("shaped_ladies") + G2.cases("shaped_saint")
    assert cases
    part = None
    saint_norms = None
    for case in cases:
        m = G2.meta[case]
        if part is None:
            part = O.partition_nodes(g.n_nodes, m["k"], "random", seed=m["pseed"])
        cfg = O.SamplerConfig(budget=m["budget"], skew_constant=m["D"], mode=m["mode"])
        rng = O.spawn_rng(m["seed"], "plan", m["epoch"], m["it"], m["worker"])
        if m["kind"] == "shaped_ladies":
            batch = shaped_batch(g, part, m)
            plan = O.ladies_plan(g, part, m["worker"], batch, cfg, m["n_layers"], rng)
        else:
            train = np.flatnonzero(g.train_mask)
            if saint_norms is None and m["mode"] != "local":
                saint_norms = O.column_norms(g, train, train)
            plan = O.saint_plan(g, part, m["worker"], train, m["budget"], cfg, m["n_layers"], rng,
                                norms=None if m["mode"] == "local" else saint_norms)
        assert_plan_equal(plan_to_dict(plan), G2.expected_plan(case))


def test_reddit_forward_backward_golden():
    """The oracle's loss_and_backward at the benchmarked configuration (Reddit shape, dims
    [602, 256 x 4, 41]) against the reference's (tests/golden/golden_reddit_fb.npz)."""
    G2 = golden("reddit_fb")
    sgph = shaped("reddit")
    assert sgph.structure_hash() == G2.meta["shape_reddit"]["structure_sha"]
    assert sgph.features_hash() == G2.meta["shape_reddit"]["features_sha"]
    g = oracle_graph_from_shaped(sgph)
    part = O.partition_nodes(g.n_nodes, 8, "random", seed=1)
    for case in G2.cases("reddit_fb"):
        m = G2.meta[case]
        batch = shaped_batch(g, part, m)
        np.testing.assert_array_equal(batch, G2.get(case, "batch"))
        plan = O.ladies_plan(g, part, m["worker"], batch,
                             O.SamplerConfig(budget=512, skew_constant=m["D"], mode=m["mode"]), 5,
                             O.spawn_rng(0, "plan", 0, 0, m["worker"]))
        np.testing.assert_array_equal(plan.remote_per_layer(), G2.get(case, "remote"))
        ws = O.init_model(m["dims"], m["model_seed"])
        loss, grads = O.loss_and_backward(ws, plan, g.features, g.labels)
        assert loss == pytest.approx(float(G2.get(case, "loss")), rel=1e-12)
        np.testing.assert_allclose(O.forward(ws, plan, g.features), G2.get(case, "logits"),
                                   rtol=1e-10, atol=1e-13)
        for l, gr in enumerate(grads):
            idx = G2.get(case, f"grad{l}_idx")
            np.testing.assert_allclose(gr.reshape(-1)[idx], G2.get(case, f"grad{l}_val"),
                                       rtol=1e-9, atol=1e-15)
            assert np.linalg.norm(gr) == pytest.approx(float(G2.get(case, f"grad{l}_norm")), rel=1e-12)


def test_reddit_pipeline_golden_plans():
    """The oracle's plans for one 24-plan look-ahead group (iterations 0..2, k = 8) at the
    Reddit shape equal the reference's (golden_pipeline.npz), a spot check of 4 plans."""
    G2 = golden("pipeline")
    m = G2.meta["pipeline"]
    sgph = shaped("reddit")
    assert sgph.structure_hash() == m["structure_sha"]
    g = oracle_graph_from_shaped(sgph)
    part = O.partition_nodes(g.n_nodes, m["k"], "random", seed=m["pseed"])
    cfg = O.SamplerConfig(budget=m["budget"], skew_constant=m["D"], mode=m["mode"])
    for it, w in ((0, 0), (1, 3), (2, 7), (2, 4)):
        meta = dict(seed=0, epoch=0, it=it, worker=w, budget=m["batch_size"])
        batch = shaped_batch(g, part, meta)
        plan = O.ladies_plan(g, part, w, batch, cfg, 5, O.spawn_rng(0, "plan", 0, it, w))
        case = f"pipe_{it}_{w}"
        np.testing.assert_array_equal(plan.batch, G2.get(case, "batch"))
        np.testing.assert_array_equal(plan.remote_per_layer(), G2.get(case, "remote"))
        for l, L in enumerate(plan.layers):
            b = L.block.tocsr()
            np.testing.assert_array_equal(L.nodes, G2.get(case, f"L{l}/nodes"))
            np.testing.assert_array_equal(b.indptr, G2.get(case, f"L{l}/indptr"))
            np.testing.assert_array_equal(b.indices, G2.get(case, f"L{l}/indices"))
            np.testing.assert_array_equal(b.data, G2.get(case, f"L{l}/data"))


GR = golden("rng")


@pytest.mark.parametrize("case", GR.cases("ladies") + GR.cases("saint"))
def test_non_pcg64_generators(case):
    """Plans driven by Philox / MT19937 / SFC64 Generators (reference accepts any Generator)."""
    m = GR.meta[case]
    g = small_graph(m["graph"])
    part = partition_for(m, g.n_nodes)
    rng = make_rng(m["rng"])
    if m["kind"] == "ladies":
        plan = O.ladies_plan(g, part, m["worker"], np.array(m["batch"], dtype=np.int64),
                             cfg_for(m), m["n_layers"], rng)
    else:
        plan = O.saint_plan(g, part, m["worker"], np.array(m["train"], dtype=np.int64), m["size"],
                            cfg_for(m), m["n_layers"], rng)
    assert_plan_equal(plan_to_dict(plan), GR.expected_plan(case))
    np.testing.assert_array_equal(rng.random(4), GR.get(case, "after"))
