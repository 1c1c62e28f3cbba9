"""The multi-GPU feature path on one device: feature rows split into per-rank shards,
gathered through the (rank, row) pointer table exactly as peers' NVLink-mapped shards
would be.  Logits and gradients must equal the single-store run bit for bit."""

import numpy as np
import pytest

import skewgcn_oracle as O

pytestmark = pytest.mark.gpu


def test_sharded_feature_gather_equals_single_store():
    import paper_2101_07706_b200 as pkg
    from paper_2101_07706_b200 import _device as D
    from paper_2101_07706_b200.training import feature_shard_map, worker_ranks

    r = np.random.default_rng(5)
    n = 2000
    e = np.stack([r.integers(0, n, 12000), r.integers(0, n, 12000)], 1)
    og = O.normalize_weights(O.graph_from_edge_array(e, n))
    X = r.normal(size=(n, 37))
    y = r.integers(0, 5, size=n)
    g = pkg.WeightedGraph(n_nodes=n, offsets=og.offsets, neighbors=og.neighbors,
                          weights=og.weights, normalized=True)
    k, world = 4, 3
    part = pkg.partition_nodes(n, k, "random", seed=2)
    cfg = pkg.SamplerConfig(budget=128, mode="skewed", skew_constant=8.0)
    model = pkg.init_model([37, 16, 16, 5], seed=1)
    for dtype in ("float64", "float32"):
        pkg.set_compute_dtype(dtype)
        plan = pkg.ladies_plan(g, part, 1, part.owned_by(1)[:100], cfg, 3, np.random.default_rng(3))
        ref_logits = pkg.forward(model, plan, X)
        ref_loss, ref_grads = pkg.loss_and_backward(model, plan, X, y)
        dg = D.device_graph(g)
        wr = worker_ranks(k, list(range(k)), world)
        node_rank, node_row, rows = feature_shard_map(part.owner, wr, world)
        ptrs = [dg.upload_shard(X[rows[rk]], dtype) for rk in range(world)]
        dg.set_feature_shards(ptrs, node_rank, node_row)
        logits = pkg.forward(model, plan, X)
        loss, grads = pkg.loss_and_backward(model, plan, X, y)
        np.testing.assert_array_equal(logits, ref_logits)
        assert loss == ref_loss
        for a, b in zip(grads, ref_grads):
            np.testing.assert_array_equal(a, b)
        dg.feat_key = None   # back to the single store for the next dtype
    pkg.set_compute_dtype("float64")
