"""Bit-packed multi-hot features and the layer-0 SpMM with the X[S_0]
gather fused in: results must equal the dense path bit for bit (the bits expand to exact
0 / 1), and the oracle (reference algorithm, fp64) within the usual tolerances."""

import numpy as np
import pytest

import skewgcn_oracle as O
from golden_util import oracle_graph_from_shaped, shaped

pytestmark = pytest.mark.gpu


def _run(P, g, part, X, dtype, monkeypatch, bits):
    monkeypatch.setenv("SKG_FEATURE_BITS", "1" if bits else "0")
    g.features = X
    ws = O.init_model([X.shape[1], 64, 64, 7], 3)
    cfg = P.SamplerConfig(budget=256, skew_constant=4.0, mode="skewed")
    batch = np.flatnonzero(g.train_mask & (part.owner == 0))[:256]
    plan = P.ladies_plan(g, part, 0, batch, cfg, 3, np.random.default_rng(11))
    P.set_compute_dtype(dtype)
    try:
        loss, grads = P.loss_and_backward(P.GcnModel([w.copy() for w in ws]), plan, X, g.labels)
        logits = P.predict_logits(P.GcnModel([w.copy() for w in ws]), g)
    finally:
        P.set_compute_dtype("float64")
    return ws, plan, loss, grads, logits


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_bit_packed_features_equal_dense(dtype, monkeypatch):
    import paper_2101_07706_b200 as P
    sg = shaped("cora")  # 1433-d bag of words: 0/1 rows
    g = P.from_shaped(sg)
    part = P.partition_nodes(sg.n_nodes, 4, "random", seed=1)
    dense = np.array(sg.features, copy=True)
    packed = P.BitFeatures.from_dense(dense)
    ws, plan, l0, g0, z0 = _run(P, g, part, dense, dtype, monkeypatch, bits=False)
    _, _, l1, g1, z1 = _run(P, g, part, packed, dtype, monkeypatch, bits=True)
    from paper_2101_07706_b200 import _device as D
    assert D.device_graph(g).xbits, "packed features were not stored bit-packed"
    assert l0 == l1
    for a, b in zip(g0, g1):
        assert np.array_equal(a, b)
    assert np.array_equal(z0, z1)
    # and the reference algorithm on the same plan
    og = oracle_graph_from_shaped(sg)
    oplan = O.ladies_plan(og, O.partition_nodes(sg.n_nodes, 4, "random", seed=1), 0,
                          np.flatnonzero(og.train_mask & (part.owner == 0))[:256],
                          O.SamplerConfig(budget=256, skew_constant=4.0, mode="skewed"), 3,
                          np.random.default_rng(11))
    ol, og_ = O.loss_and_backward(ws, oplan, og.features, og.labels)
    rtol = 1e-9 if dtype == "float64" else 1e-4
    assert abs(l1 - ol) <= rtol * abs(ol)
    for a, b in zip(g1, og_):
        np.testing.assert_allclose(a, b, rtol=rtol, atol=rtol * max(1.0, float(np.abs(b).max())))
    ref = O.predict_logits(ws, og)
    np.testing.assert_allclose(z1, ref, rtol=rtol, atol=rtol * float(np.abs(ref).max()))


def test_dense_binary_features_auto_pack():
    """A dense 0/1 matrix at least 256 wide is packed on upload (SKG_FEATURE_BITS unset)."""
    import paper_2101_07706_b200 as P
    from paper_2101_07706_b200 import _device as D
    sg = shaped("youtube_s")  # 256-d multi-hot
    g = P.from_shaped(sg)
    dg = D.device_graph(g)
    dg.ensure_features(np.array(sg.features, copy=True), "float32")
    assert dg.xbits
    dg.ensure_features(np.random.default_rng(0).normal(size=sg.features.shape).astype(np.float32), "float32")
    assert not dg.xbits
