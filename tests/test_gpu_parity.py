"""CUDA path vs the reference: golden vectors (made by the unmodified reference) and the
live CPU oracle.  Sampled node sets, block indices and ledger counts must be bit-exact;
block values within 1e-12 relative (CUDA expm1/log1p in p = -expm1(B log1p(-q)) may
differ from glibc by an ulp); q (candidate probabilities) bit-exact."""

import ctypes as C
import warnings

import numpy as np
import pytest

import skewgcn_oracle as O
from golden_util import (assert_plan_equal, cfg_for, golden, make_rng, oracle_graph_from_shaped,
                         partition_for, plan_to_dict, shaped, shaped_batch, small_graph)

pytestmark = pytest.mark.gpu

VAL_RTOL = 1e-12


def P():
    import paper_2101_07706_b200 as pkg
    return pkg


def to_pkg_graph(og):
    pkg = P()
    g = pkg.WeightedGraph(n_nodes=og.n_nodes, offsets=og.offsets, neighbors=og.neighbors,
                          weights=og.weights, normalized=True, features=og.features,
                          labels=og.labels, train_mask=og.train_mask, val_mask=og.val_mask,
                          test_mask=og.test_mask)
    return g


_GRAPHS = {}


def pkg_small_graph(name):
    if name not in _GRAPHS:
        _GRAPHS[name] = to_pkg_graph(small_graph(name))
    return _GRAPHS[name]


def pkg_partition(m, n):
    op = partition_for(m, n)
    return P().Partition(n_workers=op.n_workers, owner=op.owner)


def pkg_cfg(m):
    return P().SamplerConfig(budget=m["budget"], skew_constant=m["D"], mode=m["mode"],
                             min_scale=m.get("min_scale", 1.0))


G = golden("small")


@pytest.mark.parametrize("case", G.cases("ladies"))
def test_ladies_golden_small(case):
    m = G.meta[case]
    g = pkg_small_graph(m["graph"])
    rng = make_rng(m["rng"])
    plan = P().ladies_plan(g, pkg_partition(m, g.n_nodes), m["worker"],
                           np.array(m["batch"], dtype=np.int64), pkg_cfg(m), m["n_layers"], rng)
    assert_plan_equal(plan_to_dict(plan), G.expected_plan(case), value_rtol=VAL_RTOL)
    # the generator was advanced by exactly the uniforms the reference consumed
    ref_rng = make_rng(m["rng"])
    O.ladies_plan(small_graph(m["graph"]), partition_for(m, g.n_nodes), m["worker"],
                  np.array(m["batch"]), cfg_for(m), m["n_layers"], ref_rng)
    assert rng.bit_generator.state == ref_rng.bit_generator.state


@pytest.mark.parametrize("case", G.cases("saint"))
def test_saint_golden_small(case):
    m = G.meta[case]
    g = pkg_small_graph(m["graph"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        plan = P().saint_plan(g, pkg_partition(m, g.n_nodes), m["worker"],
                              np.array(m["train"], dtype=np.int64), m["size"], pkg_cfg(m),
                              m["n_layers"], make_rng(m["rng"]))
    assert_plan_equal(plan_to_dict(plan), G.expected_plan(case), value_rtol=VAL_RTOL)


@pytest.mark.parametrize("dtype,rtol,atol", [("float64", 1e-9, 1e-13), ("float32", 1e-4, 1e-6)])
@pytest.mark.parametrize("case", G.cases("fb"))
def test_forward_backward_golden(case, dtype, rtol, atol):
    pkg = P()
    m = G.meta[case]
    g = pkg_small_graph(m["graph"])
    plan = pkg.ladies_plan(g, pkg_partition(m, g.n_nodes), m["worker"],
                           np.array(m["batch"], dtype=np.int64), pkg_cfg(m), m["n_layers"],
                           make_rng(m["rng"]))
    x, y = G.get(case, "features"), G.get(case, "labels")
    model = pkg.init_model(m["dims"], m["model_seed"])
    old = pkg.compute_dtype()
    pkg.set_compute_dtype(dtype)
    try:
        loss, grads = pkg.loss_and_backward(model, plan, x, y)
        logits = pkg.forward(model, plan, x)
    finally:
        pkg.set_compute_dtype(old)
    scale = lambda a: atol * max(1.0, float(np.abs(a).max()))  # noqa: E731  norm-aware floor
    ref_logits = G.get(case, "logits")
    np.testing.assert_allclose(logits, ref_logits, rtol=rtol, atol=scale(ref_logits))
    assert loss == pytest.approx(float(G.get(case, "loss")), rel=rtol)
    for l, gr in enumerate(grads):
        ref = G.get(case, f"grad{l}")
        np.testing.assert_allclose(gr, ref, rtol=rtol, atol=scale(ref))


@pytest.mark.parametrize("ks", [2, 3, 4])
@pytest.mark.parametrize("case", G.cases("fb"))
def test_forward_backward_dw_ksplit(case, ks):
    """dW GEMMs with every slot's K split into ks runs (empty runs included for short
    slots), reduced in (slot, run) order: same gradients as the golden run."""
    from paper_2101_07706_b200._native import lib
    pkg = P()
    m = G.meta[case]
    g = pkg_small_graph(m["graph"])
    plan = pkg.ladies_plan(g, pkg_partition(m, g.n_nodes), m["worker"],
                           np.array(m["batch"], dtype=np.int64), pkg_cfg(m), m["n_layers"],
                           make_rng(m["rng"]))
    x, y = G.get(case, "features"), G.get(case, "labels")
    model = pkg.init_model(m["dims"], m["model_seed"])
    old = pkg.compute_dtype()
    pkg.set_compute_dtype("float32")
    lib.skg_debug_gemm_ksplit(ks)
    try:
        loss, grads = pkg.loss_and_backward(model, plan, x, y)
    finally:
        lib.skg_debug_gemm_ksplit(0)
        pkg.set_compute_dtype(old)
    assert loss == pytest.approx(float(G.get(case, "loss")), rel=1e-4)
    for l, gr in enumerate(grads):
        ref = G.get(case, f"grad{l}")
        np.testing.assert_allclose(gr, ref, rtol=1e-4, atol=1e-6 * max(1.0, float(np.abs(ref).max())))


@pytest.mark.parametrize("case", G.cases("train"))
def test_train_distributed_golden(case):
    pkg = P()
    m = G.meta[case]
    g = pkg.WeightedGraph(n_nodes=m["n"], offsets=G.get(case, "offsets"),
                          neighbors=G.get(case, "neighbors"), weights=G.get(case, "weights"),
                          normalized=True, features=G.get(case, "features"),
                          labels=G.get(case, "labels"), train_mask=G.get(case, "train_mask"),
                          val_mask=G.get(case, "val_mask"))
    part = pkg.partition_nodes(m["n"], m["k"], "random", seed=m["pseed"])
    model = pkg.init_model(m["dims"], m["model_seed"])
    cfg = pkg.SamplerConfig(budget=m["budget"], skew_constant=m["D"], mode=m["mode"])
    pkg.set_compute_dtype("float64")
    metrics, ledger = pkg.train_distributed(
        g, part, model, cfg, epochs=m["epochs"], batch_size=m["batch_size"], lr=m["lr"],
        mode=m["mode"], seed=m["seed"], sampler=m["sampler"], subgraph_size=m["subgraph_size"],
        optimizer=m["optimizer"])
    np.testing.assert_array_equal(ledger.counts, G.get(case, "ledger"))
    got = np.array([[r.epoch, r.worker, r.loss, r.train_acc, r.val_acc, r.comm_nodes_epoch]
                    for r in metrics.rows])
    np.testing.assert_allclose(got, G.get(case, "metrics"), rtol=1e-9, atol=1e-12)
    for l, w in enumerate(model.weights):
        np.testing.assert_allclose(w, G.get(case, f"w{l}"), rtol=1e-9, atol=1e-12)


def _shaped_pkg(shape):
    import torch
    sgph = shaped(shape, device="cuda" if torch.cuda.is_available() else None)
    return sgph, P().from_shaped(sgph)


@pytest.mark.parametrize("shape", ["cora", "reddit_s", "amazon_s", "reddit", "youtube", "amazon"])
def test_shaped_golden(shape):
    """Reference plans at the benchmark shapes.  YouTube (1.1M nodes > 16 x 65536) runs the
    global-atomic expand path; Amazon is the full 1.6M-node, 132M-entry GraphSAINT shape."""
    try:
        G2 = golden(shape)
    except FileNotFoundError:
        pytest.skip(f"no golden_{shape}.npz")
    pkg = P()
    gm = G2.meta[f"shape_{shape}"]
    sgph, g = _shaped_pkg(shape)
    assert sgph.structure_hash() == gm["structure_sha"], "generator drifted from the golden graph"
    cases = G2.cases("shaped_ladies") + G2.cases("shaped_saint")
    og_light = O.Graph(n_nodes=sgph.n_nodes, offsets=sgph.offsets, neighbors=sgph.neighbors,
                       weights=sgph.weights, train_mask=sgph.train_mask)
    part = None
    for case in cases:
        m = G2.meta[case]
        if part is None:
            opart = O.partition_nodes(g.n_nodes, m["k"], "random", seed=m["pseed"])
            part = pkg.Partition(n_workers=m["k"], owner=opart.owner)
        cfg = pkg.SamplerConfig(budget=m["budget"], skew_constant=m["D"], mode=m["mode"])
        rng = O.spawn_rng(m["seed"], "plan", m["epoch"], m["it"], m["worker"])
        if m["kind"] == "shaped_ladies":
            batch = shaped_batch(og_light, opart, m)
            plan = pkg.ladies_plan(g, part, m["worker"], batch, cfg, m["n_layers"], rng)
        else:
            train = np.flatnonzero(sgph.train_mask)
            plan = pkg.saint_plan(g, part, m["worker"], train, m["budget"], cfg, m["n_layers"], rng)
        assert_plan_equal(plan_to_dict(plan), G2.expected_plan(case), value_rtol=VAL_RTOL)


# --------------------------------------------------------------------- exact reductions
def _debug_reduce(a):
    from paper_2101_07706_b200._native import check, lib, ptr
    a = np.ascontiguousarray(a, dtype=np.float64)
    cdf = np.zeros_like(a)
    tot, T = C.c_double(), C.c_double()
    check(lib.skg_debug_reduce(ptr(a, C.c_double), len(a), ptr(cdf, C.c_double), C.byref(tot),
                               C.byref(T)))
    return cdf, tot.value, T.value


def _arrays():
    r = np.random.default_rng(0)
    yield "uniform-154k", r.random(154_321) + 1e-3
    yield "lognormal-1.36M", np.exp(r.normal(size=1_360_000) * 2)
    yield "ties", (r.integers(1, 2 ** 20, size=200_000) * 2.0 ** -60)  # many exact .5-ulp ties
    yield "huge-first", np.concatenate([[1e6], r.random(50_000)])
    yield "huge-middle", np.concatenate([r.random(30_000), [1e9], r.random(30_000)])
    yield "tiny-tail", np.concatenate([r.random(1000), np.full(100_000, 1e-30)])
    yield "mixed-scales", r.random(300_000) * 10.0 ** r.integers(-12, 3, size=300_000)
    yield "two", np.array([0.3, 0.7])
    yield "len-129", r.random(129)
    yield "len-8191", r.random(8191)
    for n in (1000, 1025, 4096, 33_000, 65_537):
        yield f"n{n}", r.random(n) ** 4


@pytest.mark.parametrize("name,a", list(_arrays()), ids=lambda x: x if isinstance(x, str) else "")
def test_exact_cumsum_and_pairwise(name, a):
    cdf, total, T = _debug_reduce(a)
    assert total == a.sum(), "pairwise sum differs from numpy"
    ref = np.cumsum(a)
    assert T == ref[-1]
    mism = np.flatnonzero(cdf != ref)
    assert len(mism) == 0, f"{len(mism)} cumsum mismatches, first at {mism[:5]}"


# --------------------------------------------------------------------- live oracle
@pytest.mark.parametrize("seed", range(6))
def test_random_plans_vs_oracle(seed):
    pkg = P()
    r = np.random.default_rng(100 + seed)
    n = int(r.integers(300, 3000))
    deg = float(r.uniform(3, 40))
    m = int(n * deg / 2)
    u = r.integers(0, n, m)
    v = r.integers(0, n, m)
    e = np.stack([u[u != v], v[u != v]], 1)
    og = O.normalize_weights(O.graph_from_edge_array(e, n))
    g = to_pkg_graph(og)
    k = int(r.integers(1, 9))
    opart = O.partition_nodes(n, k, "random", seed=seed)
    part = pkg.Partition(n_workers=k, owner=opart.owner)
    for mode in ("full", "skewed", "local"):
        w = int(r.integers(0, k))
        owned = opart.owned_by(w)
        if len(owned) == 0:
            continue
        batch = owned[: int(r.integers(1, 200))]
        B = int(r.integers(1, 600))
        D = float(r.choice([0.0, 4.0, 8.0, 16.0, 32.0]))
        L = int(r.integers(1, 6))
        ocfg = O.SamplerConfig(budget=B, skew_constant=D, mode=mode)
        cfg = pkg.SamplerConfig(budget=B, skew_constant=D, mode=mode)
        exp = O.ladies_plan(og, opart, w, batch, ocfg, L, np.random.default_rng(seed))
        got = pkg.ladies_plan(g, part, w, batch, cfg, L, np.random.default_rng(seed))
        assert_plan_equal(plan_to_dict(got), plan_to_dict(exp), value_rtol=VAL_RTOL)
        train = np.sort(r.choice(n, size=int(r.integers(2, n)), replace=False))
        sub = int(r.integers(1, len(train) + 1))
        norms = O.column_norms(og, train, train) if mode != "local" else None
        try:
            exp_s = O.saint_plan(og, opart, w, train, sub, ocfg, 2, np.random.default_rng(seed),
                                 norms=norms)
        except ValueError:
            with pytest.raises(ValueError):
                pkg.saint_plan(g, part, w, train, sub, cfg, 2, np.random.default_rng(seed))
            continue
        got_s = pkg.saint_plan(g, part, w, train, sub, cfg, 2, np.random.default_rng(seed))
        assert_plan_equal(plan_to_dict(got_s), plan_to_dict(exp_s), value_rtol=VAL_RTOL)


# --------------------------------------------------------------------- reference behaviours
def test_errors_match_reference():
    pkg = P()
    g = pkg_small_graph("er20")
    part = pkg.partition_nodes(20, 1, "contiguous")
    cfg = pkg.SamplerConfig(budget=21, mode="full")
    with pytest.raises(ValueError):
        pkg.ladies_plan(g, part, 0, np.array([], dtype=np.int64), cfg, 2, np.random.default_rng(0))
    plan = pkg.ladies_plan(g, part, 0, np.arange(3), cfg, 1, np.random.default_rng(0))
    model = pkg.init_model([4, 3], seed=0)
    x = np.random.default_rng(0).normal(size=(20, 4))
    with pytest.raises(ValueError, match="labeled"):
        pkg.loss_and_backward(model, plan, x, np.full(20, -1))
    with pytest.raises(ValueError, match="depth"):
        pkg.forward(pkg.init_model([4, 3, 3], seed=0), plan, x)
    with pytest.warns(UserWarning, match="clamping"):
        pkg.saint_plan(g, part, 0, np.arange(20), 30, cfg, 1, np.random.default_rng(0))


def test_saturated_forward_equals_full_graph():
    pkg = P()
    og = small_graph("er20")
    g = to_pkg_graph(og)
    rng = np.random.default_rng(501)
    X = rng.normal(size=(20, 4))
    g.features = X
    part = pkg.partition_nodes(20, 2, "contiguous")
    model = pkg.init_model([4, 6, 3], seed=2)
    batch = part.owned_by(0)[:5]
    plan = pkg.ladies_plan(g, part, 0, batch, pkg.SamplerConfig(budget=21, mode="full"), 2,
                           np.random.default_rng(1))
    pkg.set_compute_dtype("float64")
    sampled = pkg.forward(model, plan, X)
    exact = pkg.predict_logits(model, g)[batch]
    np.testing.assert_allclose(sampled, exact, atol=1e-10)
    ref = O.predict_logits(model.weights, O.Graph(20, og.offsets, og.neighbors, og.weights,
                                                  features=X))[batch]
    np.testing.assert_allclose(exact, ref, rtol=1e-10, atol=1e-12)


def test_device_graph_queries():
    pkg = P()
    og = small_graph("er60")
    g = to_pkg_graph(og)
    s = np.array([1, 5, 9, 33])
    np.testing.assert_array_equal(pkg.neighbor_union(g, s), O.neighbor_union(og, s))
    c = O.neighbor_union(og, s)
    np.testing.assert_array_equal(pkg.column_norms(g, s, c), O.column_norms(og, s, c))
    cols = np.array([0, 1, 2, 5, 7, 33, 50])
    a = pkg.adjacency_block(g, s, cols).toarray()
    b = O.adjacency_block(og, s, cols).toarray()
    np.testing.assert_array_equal(a, b)
    with pytest.raises(ValueError, match="not adjacent"):
        pkg.column_norms(g, s, np.array([int(np.setdiff1d(np.arange(60), c)[0])]))


def test_kernel_launch_counter_moves():
    pkg = P()
    before = pkg.kernel_launches()
    g = pkg_small_graph("er30")
    pkg.ladies_plan(g, pkg.partition_nodes(30, 2, "hash"), 0, np.arange(0, 30, 3),
                    pkg.SamplerConfig(budget=5, mode="skewed", skew_constant=4.0), 3,
                    np.random.default_rng(0))
    assert pkg.kernel_launches() > before


@pytest.mark.parametrize("seed", range(3))
def test_unnormalised_asymmetric_graph_vs_oracle(seed):
    """Arbitrary positive weights (not 1/sqrt(d_i d_j), not symmetric): the stored-weight
    bucket path and the transposed (CSC) pull-norm path."""
    pkg = P()
    r = np.random.default_rng(700 + seed)
    n = 800
    m = 6000
    u, v = r.integers(0, n, m), r.integers(0, n, m)
    og = O.normalize_weights(O.graph_from_edge_array(np.stack([u, v], 1), n))
    og.weights = r.uniform(0.05, 2.0, size=len(og.weights))   # break normalisation and symmetry
    g = to_pkg_graph(og)
    k = 3
    opart = O.partition_nodes(n, k, "random", seed=seed)
    part = pkg.Partition(n_workers=k, owner=opart.owner)
    for mode, D in (("full", 0.0), ("skewed", 8.0), ("local", 0.0)):
        ocfg = O.SamplerConfig(budget=64, skew_constant=D, mode=mode)
        cfg = pkg.SamplerConfig(budget=64, skew_constant=D, mode=mode)
        batch = opart.owned_by(1)[:50]
        exp = O.ladies_plan(og, opart, 1, batch, ocfg, 3, np.random.default_rng(seed))
        got = pkg.ladies_plan(g, part, 1, batch, cfg, 3, np.random.default_rng(seed))
        assert_plan_equal(plan_to_dict(got), plan_to_dict(exp), value_rtol=VAL_RTOL)
        train = np.sort(r.choice(n, 300, replace=False))
        norms = O.column_norms(og, train, train) if mode != "local" else None
        exp_s = O.saint_plan(og, opart, 1, train, 40, ocfg, 2, np.random.default_rng(seed), norms=norms)
        got_s = pkg.saint_plan(g, part, 1, train, 40, cfg, 2, np.random.default_rng(seed))
        assert_plan_equal(plan_to_dict(got_s), plan_to_dict(exp_s), value_rtol=VAL_RTOL)


@pytest.mark.parametrize("normalised", [True, False])
def test_dense_graph_heavy_contributions_vs_oracle(normalised):
    """Dense graph: candidates receive up to ~100 contributions, so the light slots (<= 4),
    the 8-lane and warp heavy folds (5..32) and the CTA fold (> 32) all run; with stored
    (non-normalised, asymmetric) weights the slot/overflow weight copies are used too."""
    pkg = P()
    r = np.random.default_rng(4242 + int(normalised))
    n = 400
    m = 40000
    u, v = r.integers(0, n, m), r.integers(0, n, m)
    og = O.normalize_weights(O.graph_from_edge_array(np.stack([u, v], 1), n))
    if not normalised:
        og.weights = r.uniform(0.05, 2.0, size=len(og.weights))
    g = to_pkg_graph(og)
    k = 2
    opart = O.partition_nodes(n, k, "random", seed=3)
    part = pkg.Partition(n_workers=k, owner=opart.owner)
    for mode, D in (("full", 0.0), ("skewed", 8.0), ("local", 0.0)):
        for budget in (16, 128):
            ocfg = O.SamplerConfig(budget=budget, skew_constant=D, mode=mode)
            cfg = pkg.SamplerConfig(budget=budget, skew_constant=D, mode=mode)
            batch = opart.owned_by(0)[:180]
            exp = O.ladies_plan(og, opart, 0, batch, ocfg, 3, np.random.default_rng(11))
            got = pkg.ladies_plan(g, part, 0, batch, cfg, 3, np.random.default_rng(11))
            assert_plan_equal(plan_to_dict(got), plan_to_dict(exp), value_rtol=VAL_RTOL)


def test_column_norms_pull_large_row_set_vs_oracle():
    """column_norms over a large row set (> the push path's limit) uses the pull
    formulation; it must equal the oracle's np.add.at fold bit for bit, and raise the
    reference's error for non-adjacent candidates."""
    pkg = P()
    r = np.random.default_rng(99)
    n, m = 30000, 150000
    u, v = r.integers(0, n, m), r.integers(0, n, m)
    og = O.normalize_weights(O.graph_from_edge_array(np.stack([u, v], 1), n))
    g = to_pkg_graph(og)
    rows = np.sort(r.choice(n, 20000, replace=False))
    cand = O.neighbor_union(og, rows)
    exp = O.column_norms(og, rows, cand)
    got = pkg.column_norms(g, rows, cand)
    assert np.array_equal(got, exp)
    isolated = np.setdiff1d(np.arange(n), cand)
    if len(isolated):
        with pytest.raises(ValueError, match="not adjacent"):
            pkg.column_norms(g, rows, np.sort(np.concatenate([cand[:5], isolated[:1]])))


GR = golden("rng")


@pytest.mark.parametrize("case", GR.cases("ladies") + GR.cases("saint"))
def test_non_pcg64_generators(case):
    """Philox4x64-10 streams generated on the device (fresh and part-used output buffers)
    and explicit uniforms from MT19937 / SFC64 Generators: plans bit-exact with the
    reference's, and the caller's generator left where the reference leaves it."""
    m = GR.meta[case]
    g = pkg_small_graph(m["graph"])
    part = pkg_partition(m, g.n_nodes)
    rng = make_rng(m["rng"])
    if m["kind"] == "ladies":
        plan = P().ladies_plan(g, part, m["worker"], np.array(m["batch"], dtype=np.int64),
                               pkg_cfg(m), m["n_layers"], rng)
    else:
        plan = P().saint_plan(g, part, m["worker"], np.array(m["train"], dtype=np.int64),
                              m["size"], pkg_cfg(m), m["n_layers"], rng)
    assert_plan_equal(plan_to_dict(plan), GR.expected_plan(case), value_rtol=VAL_RTOL)
    np.testing.assert_array_equal(rng.random(4), GR.get(case, "after"))


def test_philox_device_stream_many_blocks():
    """A Reddit-sized draw count: Philox outputs far past the first counter block (and a
    counter carry across the low word) equal numpy's on every sampled layer."""
    og = O.normalize_weights(O.graph_from_edge_array(
        np.stack(np.triu_indices(400, 1), 1)[np.random.default_rng(1).random(79800) < 0.05], 400))
    g = to_pkg_graph(og)
    part = O.partition_nodes(400, 4, "random", seed=2)
    ppart = P().Partition(n_workers=4, owner=part.owner)
    batch = part.owned_by(1)[:60]
    for key, skip in ((5, 0), (2**64 - 1, 2)):
        bg = np.random.Philox(key=key)
        st = bg.state
        st["state"]["counter"] = np.array([2**64 - 3, 2**64 - 1, 0, 0], dtype=np.uint64)
        bg.state = st
        bg.random_raw(skip)
        st = bg.state
        rng_o = np.random.Generator(np.random.Philox(key=key))
        rng_d = np.random.Generator(np.random.Philox(key=key))
        rng_o.bit_generator.state = st
        rng_d.bit_generator.state = st
        exp = O.ladies_plan(og, part, 1, batch, O.SamplerConfig(budget=48, skew_constant=8.0), 5,
                            rng_o)
        got = P().ladies_plan(g, ppart, 1, batch, P().SamplerConfig(budget=48, skew_constant=8.0),
                              5, rng_d)
        assert_plan_equal(plan_to_dict(got), plan_to_dict(exp), value_rtol=VAL_RTOL)
        np.testing.assert_array_equal(rng_d.random(4), rng_o.random(4))
