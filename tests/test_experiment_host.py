"""Experiment configs, dataset formats and the block-model generator (CPU): against the
reference's own outputs frozen by tests/golden/make_golden_experiment.py."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2101_07706_b200 as P
from paper_2101_07706_b200.datasets import load_edge_list, save_edge_list

GOLD = Path(__file__).parent / "golden" / "experiment"
CASES = ["tiny", "ladies_adam", "saint"]


def _raw(case):
    return json.loads((GOLD / f"{case}.config.json").read_text())


@pytest.mark.parametrize("case", CASES)
def test_config_round_trip_matches_reference_summary(case, tmp_path):
    raw = {**_raw(case), "output_dir": str(tmp_path / "o")}
    cfg = P.ExperimentConfig.from_dict(raw)
    ref = json.loads((GOLD / case / "summary.json").read_text())["config"]
    mine = cfg.to_dict()
    assert {k: v for k, v in mine.items() if k != "output_dir"} == \
           {k: v for k, v in ref.items() if k != "output_dir"}
    P.save_config(cfg, tmp_path / "c.json")
    assert P.load_config(tmp_path / "c.json").to_dict() == mine


@pytest.mark.parametrize("bad,msg", [
    ({"dataset": {"synthetic": {}}, "bogus": 1}, "unknown config key"),
    ({"workers": 2}, "needs a 'dataset' section"),
    ({"dataset": {"path": "x", "synthetic": {"n_nodes": 4, "n_blocks": 1, "p_in": 0.5, "p_out": 0.1,
                                              "feature_dim": 2}}}, "exactly one"),
    ({"dataset": {"path": "x"}, "modes": ["skewed"]}, "needs skew_constants"),
    ({"dataset": {"path": "x"}, "modes": ["warp"]}, "unknown mode"),
    ({"dataset": {"path": "x"}, "sampler": {"kind": "saint"}}, "needs subgraph_size"),
    ({"dataset": {"path": "x"}, "epochs": 0}, "counts must be >= 1"),
    ({"dataset": {"path": "x"}, "partition": {"strategy": "random", "x": 1}}, "unknown config key"),
])
def test_config_errors(bad, msg):
    with pytest.raises((ValueError, TypeError), match=msg):
        P.ExperimentConfig.from_dict(bad)


@pytest.mark.parametrize("case", CASES)
def test_synth_sbm_is_the_reference_graph(case):
    ref = np.load(GOLD / f"sbm_{case}.npz")
    g = P.synth_sbm(P.SbmSpec(**_raw(case)["dataset"]["synthetic"]))
    for k, v in (("offsets", g.offsets), ("neighbors", g.neighbors), ("weights", g.weights),
                 ("features", g.features), ("labels", g.labels), ("train", g.train_mask),
                 ("val", g.val_mask), ("test", g.test_mask)):
        assert np.array_equal(np.asarray(v), ref[k]), k


def test_dataset_directory_round_trip(tmp_path):
    spec = P.SbmSpec(**_raw("ladies_adam")["dataset"]["synthetic"])
    P.save_dataset(P.synth_sbm(spec, normalize=False), tmp_path)
    g = P.load_dataset(tmp_path)
    ref = np.load(GOLD / "sbm_ladies_adam.npz")
    assert np.array_equal(g.offsets, ref["offsets"]) and np.array_equal(g.weights, ref["weights"])
    assert np.array_equal(g.features, ref["features"]) and np.array_equal(g.labels, ref["labels"])
    assert np.array_equal(g.test_mask, ref["test"])


@pytest.mark.parametrize("text,msg", [
    ("0 1\n1 2 3\n", ":2: expected 'u v'"),
    ("# c\n0 x\n", ":2: non-integer node id"),
    ("0 1\n\n2 -1\n", ":3: negative node id"),
])
def test_edge_list_errors(tmp_path, text, msg):
    p = tmp_path / "e.txt"
    p.write_text(text)
    with pytest.raises(ValueError, match=msg):
        load_edge_list(p)


def test_edge_list_round_trip(tmp_path):
    g = P.synth_sbm(P.SbmSpec(**_raw("tiny")["dataset"]["synthetic"]), normalize=False)
    save_edge_list(g, tmp_path / "e.txt")
    h = load_edge_list(tmp_path / "e.txt", n_hint=g.n_nodes)
    assert np.array_equal(h.offsets, g.offsets) and np.array_equal(h.neighbors, g.neighbors)


def test_partition_csv(tmp_path):
    p = tmp_path / "p.csv"
    p.write_text("node,worker\n0,1\n1,0\n2,1\n")
    part = P.load_partition_csv(p, 3, 2)
    assert part.owner.tolist() == [1, 0, 1]
    p.write_text("0,1\n2,1\n")
    with pytest.raises(ValueError, match="misses nodes"):
        P.load_partition_csv(p, 3, 2)


def test_partition_csv_errors_in_file_order(tmp_path):
    """partition.py:77-98: rows are checked as they are read; the message carries the line."""
    p = tmp_path / "p.csv"
    p.write_text("node,worker\n0,1\n7,0\nbad\n")
    with pytest.raises(ValueError, match=r"p\.csv:3: node 7 out of range"):
        P.load_partition_csv(p, 3, 2)
    p.write_text("0,1\n1,5\n")
    with pytest.raises(ValueError, match=r"p\.csv:2: worker 5 out of range"):
        P.load_partition_csv(p, 3, 2)
