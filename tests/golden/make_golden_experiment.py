"""Freeze the UNMODIFIED reference's experiment outputs for the parity tests (run in the
build container, where the reference is importable):

    python tests/golden/make_golden_experiment.py

Writes tests/golden/experiment/<case>/ (the reference's run_experiment files for the
configs in CASES) and tests/golden/experiment/sbm_<case>.npz (the reference synth_sbm
graph of each case's dataset, to pin this package's generator on CPU).
"""

from __future__ import annotations

import json
import shutil
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent / "experiment"
sys.path.insert(0, "/root/reference/pkg/src")

import skewgcn as sg  # noqa: E402  (reference, read-only)

CASES = {
    # the reference test-suite's tiny grid (test_experiment.py:16-31): all modes, two D
    "tiny": {
        "dataset": {"synthetic": {"n_nodes": 60, "n_blocks": 2, "p_in": 0.25, "p_out": 0.05,
                                  "feature_dim": 6, "noise_sigma": 0.4, "seed": 3}},
        "workers": 2, "partition": {"strategy": "random", "seed": 1},
        "sampler": {"kind": "ladies", "budget": 8}, "modes": ["full", "local", "skewed"],
        "skew_constants": [4.0, 8.0], "model": {"hidden": [8]}, "lr": 0.2, "epochs": 2,
        "batch_size": 8, "seed": 5,
    },
    # a larger LADIES grid with a deeper model and Adam
    "ladies_adam": {
        "dataset": {"synthetic": {"n_nodes": 240, "n_blocks": 4, "p_in": 0.12, "p_out": 0.01,
                                  "feature_dim": 12, "noise_sigma": 0.5, "seed": 11}},
        "workers": 4, "partition": {"strategy": "random", "seed": 2},
        "sampler": {"kind": "ladies", "budget": 24}, "modes": ["full", "skewed"],
        "skew_constants": [2.0, 16.0], "model": {"hidden": [16, 16]}, "optimizer": "adam",
        "lr": 0.01, "epochs": 3, "batch_size": 20, "seed": 7,
    },
    # GraphSAINT cells
    "saint": {
        "dataset": {"synthetic": {"n_nodes": 200, "n_blocks": 3, "p_in": 0.1, "p_out": 0.01,
                                  "feature_dim": 8, "noise_sigma": 0.3, "seed": 4}},
        "workers": 3, "partition": {"strategy": "contiguous", "seed": 0},
        "sampler": {"kind": "saint", "budget": 30, "subgraph_size": 40},
        "modes": ["full", "local", "skewed"], "skew_constants": [8.0],
        "model": {"hidden": [12]}, "lr": 0.1, "epochs": 2, "batch_size": 16, "seed": 9,
    },
}


def main() -> None:
    HERE.mkdir(parents=True, exist_ok=True)
    for name, raw in CASES.items():
        out = HERE / name
        if out.exists():
            shutil.rmtree(out)
        cfg = sg.ExperimentConfig.from_dict({**raw, "output_dir": str(out)})
        sg.run_experiment(cfg)
        (HERE / f"{name}.config.json").write_text(json.dumps(raw, indent=2, sort_keys=True) + "\n")
        g = sg.synth_sbm(sg.SbmSpec(**raw["dataset"]["synthetic"]))
        np.savez_compressed(HERE / f"sbm_{name}.npz", offsets=g.offsets, neighbors=g.neighbors,
                            weights=g.weights, features=g.features, labels=g.labels,
                            train=g.train_mask, val=g.val_mask, test=g.test_mask)
        print("wrote", out)


if __name__ == "__main__":
    main()
