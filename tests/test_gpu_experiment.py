"""run_experiment on the device path against the reference's own output files
(tests/golden/experiment, from tests/golden/make_golden_experiment.py), fp64 compute:
same files, identical integer outputs (communicated nodes, reductions), float outputs to
fp64 rounding."""

import csv
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden" / "experiment"


def _rows(path):
    with open(path) as fh:
        return list(csv.DictReader(fh))


@pytest.mark.parametrize("case", ["tiny", "ladies_adam", "saint"])
def test_run_experiment_matches_reference_outputs(case, tmp_path):
    import paper_2101_07706_b200 as P
    raw = json.loads((GOLD / f"{case}.config.json").read_text())
    prev = P.compute_dtype()
    P.set_compute_dtype("float64")
    try:
        P.run_experiment(P.ExperimentConfig.from_dict({**raw, "output_dir": str(tmp_path)}))
    finally:
        P.set_compute_dtype(prev)
    ref_dir = GOLD / case
    assert sorted(p.name for p in tmp_path.iterdir()) == sorted(p.name for p in ref_dir.iterdir())
    assert json.loads((tmp_path / "comparison.json").read_text()) == \
           json.loads((ref_dir / "comparison.json").read_text())
    got, ref = (json.loads((d / "summary.json").read_text()) for d in (tmp_path, ref_dir))
    got["config"].pop("output_dir")
    ref["config"].pop("output_dir")
    assert got["config"] == ref["config"] and got["reduction_factors"] == ref["reduction_factors"]
    for a, b in zip(got["cells"], ref["cells"]):
        for k in ("mode", "skew_constant", "total_comm_nodes", "metrics_csv"):
            assert a[k] == b[k], (k, a[k], b[k])
        for k in ("best_val_acc", "final_val_acc", "test_acc"):
            assert a[k] == pytest.approx(b[k], abs=1e-12), (k, a[k], b[k])
        ga, rb = _rows(tmp_path / a["metrics_csv"]), _rows(ref_dir / b["metrics_csv"])
        assert len(ga) == len(rb)
        for x, y in zip(ga, rb):
            for k in ("epoch", "worker", "comm_nodes_epoch", "train_acc", "val_acc"):
                assert x[k] == y[k] if k in ("epoch", "worker", "comm_nodes_epoch") else \
                    float(x[k]) == pytest.approx(float(y[k]), abs=1e-12), (k, x, y)
            assert float(x["loss"]) == pytest.approx(float(y["loss"]), rel=1e-9, abs=1e-12)
