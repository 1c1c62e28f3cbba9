"""Load the reference-generated golden vectors and rebuild their inputs."""

from __future__ import annotations

import functools
import json
from pathlib import Path

import numpy as np

import skewgcn_oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"


class Golden:
    def __init__(self, name):
        path = GOLDEN / f"golden_{name}.npz"
        self.z = np.load(path, allow_pickle=False)
        self.meta = json.loads(str(self.z["__meta__"]))

    def get(self, case, key):
        return self.z[f"{case}/{key}"]

    def has(self, case, key):
        return f"{case}/{key}" in self.z.files

    def cases(self, kind):
        return [c for c, m in self.meta.items() if isinstance(m, dict) and m.get("kind") == kind]

    def expected_plan(self, case):
        """Dict form of a golden plan: per-layer nodes / CSR / dist digests."""
        out = {"batch": self.get(case, "batch"), "remote": self.get(case, "remote"),
               "starvation": int(self.get(case, "starvation")), "layers": []}
        l = 0
        while self.has(case, f"L{l}/nodes"):
            L = {k: self.get(case, f"L{l}/{k}") for k in
                 ("nodes", "indptr", "indices", "data", "shape", "has_dist")}
            for k in ("n_cand", "q_sha", "cand_sha", "s_used", "q", "cand"):
                if self.has(case, f"L{l}/{k}"):
                    L[k] = self.get(case, f"L{l}/{k}")
            out["layers"].append(L)
            l += 1
        return out


@functools.lru_cache(maxsize=None)
def golden(name):
    return Golden(name)


@functools.lru_cache(maxsize=None)
def small_graph(name):
    g = golden("small")
    e = g.get("graph_" + name, "edges")
    n = int(g.get("graph_" + name, "n"))
    return O.normalize_weights(O.graph_from_edge_array(e, n))


@functools.lru_cache(maxsize=4)
def shaped(shape, device=None, with_features=None):
    """The benchmark-shaped graph; plan-only checks of the large shapes skip the features
    (YouTube's would be 9 GB)."""
    from paper_2101_07706_b200.synth import make_shaped_graph
    if with_features is None:
        with_features = shape not in ("youtube", "amazon")
    sg = make_shaped_graph(shape, seed=0, device=device, with_features=with_features)
    return sg


def oracle_graph_from_shaped(sgph):
    return O.Graph(n_nodes=sgph.n_nodes, offsets=sgph.offsets,
                   neighbors=sgph.neighbors.astype(np.int64), weights=sgph.weights,
                   normalized=True,
                   features=sgph.features.astype(np.float64) if sgph.features.shape[1] else None,
                   labels=sgph.labels if np.ndim(sgph.labels) == 1 else None, train_mask=sgph.train_mask, val_mask=sgph.val_mask,
                   test_mask=sgph.test_mask)


def partition_for(meta, n):
    if meta.get("strategy") == "explicit":
        return O.Partition(meta["k"], np.asarray(meta["owner"], dtype=np.int64))
    return O.partition_nodes(n, meta["k"], meta.get("strategy", "random"), seed=meta.get("pseed"))


def make_rng(spec):
    """Same construction as tests/golden/make_golden.py:make_rng."""
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
    return O.spawn_rng(spec[1], *spec[2:])


def cfg_for(meta):
    return O.SamplerConfig(budget=meta["budget"], skew_constant=meta["D"], mode=meta["mode"],
                           min_scale=meta.get("min_scale", 1.0))


def shaped_batch(g, part, meta):
    wt = np.flatnonzero(g.train_mask & (part.owner == meta["worker"]))
    take = min(meta["budget"], len(wt))
    brng = O.spawn_rng(meta["seed"], "batch", meta["epoch"], meta["it"], meta["worker"])
    return O.node_set(brng.choice(wt, size=take, replace=False))


def plan_to_dict(plan):
    """Normalise an oracle / drop-in plan into the golden dict form."""
    out = {"batch": np.asarray(plan.batch), "remote": np.asarray(plan.remote_per_layer()),
           "starvation": int(plan.starvation_events), "layers": []}
    for L in plan.layers:
        b = L.block.tocsr()
        d = {"nodes": np.asarray(L.nodes), "indptr": b.indptr.astype(np.int64),
             "indices": b.indices.astype(np.int64), "data": np.asarray(b.data),
             "shape": np.array(b.shape, dtype=np.int64), "has_dist": int(L.dist is not None)}
        if L.dist is not None:
            d["q"] = np.asarray(L.dist.q)
            d["cand"] = np.asarray(L.dist.candidates)
            d["s_used"] = float(L.dist.s_used)
        out["layers"].append(d)
    return out


def sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def assert_plan_equal(got, exp, *, value_rtol=0.0, check_dist=True):
    """Bit-exact ids / indices / ledger; block values exact or at value_rtol."""
    np.testing.assert_array_equal(got["batch"], exp["batch"])
    np.testing.assert_array_equal(got["remote"], exp["remote"])
    assert got["starvation"] == exp["starvation"]
    assert len(got["layers"]) == len(exp["layers"])
    for l, (a, b) in enumerate(zip(got["layers"], exp["layers"])):
        np.testing.assert_array_equal(a["nodes"], b["nodes"], err_msg=f"layer {l} nodes")
        np.testing.assert_array_equal(a["shape"], b["shape"], err_msg=f"layer {l} shape")
        np.testing.assert_array_equal(a["indptr"], b["indptr"], err_msg=f"layer {l} indptr")
        np.testing.assert_array_equal(a["indices"], b["indices"], err_msg=f"layer {l} indices")
        if value_rtol == 0.0:
            np.testing.assert_array_equal(a["data"], b["data"], err_msg=f"layer {l} data")
        else:
            np.testing.assert_allclose(a["data"], b["data"], rtol=value_rtol, atol=0,
                                       err_msg=f"layer {l} data")
        assert int(a["has_dist"]) == int(b["has_dist"])
        if check_dist and int(b["has_dist"]):
            if "q" in b:
                np.testing.assert_array_equal(a["q"], b["q"], err_msg=f"layer {l} q")
                np.testing.assert_array_equal(a["cand"], b["cand"])
            else:
                assert sha(np.asarray(a["q"], dtype=np.float64)) == str(b["q_sha"]), f"layer {l} q"
                assert sha(np.asarray(a["cand"], dtype=np.int64)) == str(b["cand_sha"])
            assert float(a["s_used"]) == float(b["s_used"])
