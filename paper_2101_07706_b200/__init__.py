"""B200-native skewed layer-wise sampling for distributed GCN training (arXiv 2101.07706).

A drop-in for the reference simulator's hot path (``skewgcn``): same function names,
arguments, return types and exceptions, with sampling, GCN compute and the gradient
step running as sm_100a CUDA kernels in ``libskg.so`` (see include/skewgcn_b200.h).
Importing this package requires the built library; there is no CPU fallback.
"""

from ._native import kernel_launches, lib as _lib  # noqa: F401  (fails loudly if missing)
from ._device import compute_dtype, set_compute_dtype
from .features import BitFeatures
from .graph import (WeightedGraph, adjacency_block, column_norms, from_shaped, graph_from_edges,
                    load_edge_list, neighbor_union, node_set, normalize_weights, undirected_edges)
from .partition import Partition, partition_nodes
from .sampling import ProbDist, SampleDraw, SamplerConfig
from .seeding import pcg64_state, spawn_rng
from .datasets import (SbmSpec, load_dataset, load_features_csv, load_labels_csv, load_masks_csv,
                       load_partition_csv, save_dataset, synth_sbm)
from .experiment import DatasetSpec, ExperimentConfig, load_config, run_experiment, save_config
from .training import (CommLedger, EvalResult, GcnModel, Metrics, MetricRow, PlanLayer, SamplePlan,
                       Trainer, evaluate, forward, init_model, ladies_plan, loss_and_backward,
                       predict_logits, saint_plan, train_column_norms, train_distributed)

__version__ = "0.1.0"

__all__ = [
    "BitFeatures", "WeightedGraph", "adjacency_block", "column_norms", "neighbor_union", "node_set",
    "normalize_weights", "graph_from_edges", "load_edge_list", "undirected_edges", "from_shaped",
    "Partition", "partition_nodes", "ProbDist", "SampleDraw", "SamplerConfig", "spawn_rng",
    "pcg64_state", "CommLedger", "EvalResult", "GcnModel", "Metrics", "MetricRow", "PlanLayer",
    "SamplePlan", "Trainer", "evaluate", "forward", "init_model", "ladies_plan",
    "loss_and_backward", "predict_logits", "saint_plan", "train_column_norms",
    "train_distributed", "set_compute_dtype", "compute_dtype", "kernel_launches",
    "SbmSpec", "synth_sbm", "load_dataset", "save_dataset", "load_features_csv", "load_labels_csv",
    "load_masks_csv", "load_partition_csv", "DatasetSpec", "ExperimentConfig", "load_config",
    "save_config", "run_experiment",
]
