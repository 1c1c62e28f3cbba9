"""The tensor-core GEMM's TMA-store epilogue (gemm_tc.cu: each 32-column box of the tile staged
in the idle stage ring and written by a TMA tensor store) against the per-row store epilogue
(SKG_GEMM_TMA_STORE=0): fp32 training runs whose GEMMs have ragged row tiles (per-plan M below
the launch's M), a partial last N tile (hidden 160 = 128 + 32) and a 3-class head must give
bit-identical losses, ledgers and weights.  Each variant runs in its own process because the
switch is read once per process."""

import os
import pickle
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

_RUN = r"""
import pickle, sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_2101_07706_b200 as P
P.set_compute_dtype("float32")
g = P.synth_sbm(P.SbmSpec(n_nodes=900, n_blocks=3, p_in=0.05, p_out=0.005, feature_dim=36,
                          noise_sigma=0.5, seed=7))
part = P.partition_nodes(g.n_nodes, 4, "random", seed=2)
out = []
for sampler in ("ladies", "saint"):
    model = P.init_model([36, 160, 160, 3], 4)
    metrics, ledger = P.train_distributed(
        g, part, model, P.SamplerConfig(budget=200, skew_constant=8.0, mode="skewed"),
        epochs=2, batch_size=60, lr=0.2, mode="skewed", seed=3, sampler=sampler,
        subgraph_size=150 if sampler == "saint" else None)
    out.append(([(r.epoch, r.worker, r.loss, r.comm_nodes_epoch) for r in metrics.rows],
                ledger.counts, [np.asarray(w) for w in model.weights]))
pickle.dump(out, open({path!r}, "wb"))
"""


def _run(tmp_path, tma):
    path = str(tmp_path / f"run_{tma}.pkl")
    env = dict(os.environ, SKG_GEMM_TMA_STORE=str(tma))
    r = subprocess.run([sys.executable, "-c", _RUN.format(root=str(ROOT), path=path)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return pickle.load(open(path, "rb"))


def test_tma_store_epilogue_equals_row_stores(tmp_path):
    rows_store = _run(tmp_path, 0)
    tma_store = _run(tmp_path, 1)
    assert len(rows_store) == len(tma_store) == 2
    for (rows_a, led_a, w_a), (rows_b, led_b, w_b) in zip(rows_store, tma_store):
        assert rows_a == rows_b  # losses bit-identical
        np.testing.assert_array_equal(led_a, led_b)
        for a, b in zip(w_a, w_b):
            np.testing.assert_array_equal(a, b)
        assert all(np.isfinite(r[2]) for r in rows_a)
