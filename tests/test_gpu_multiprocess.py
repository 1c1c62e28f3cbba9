"""train_distributed with one process per rank (gloo, ranks sharing the test box's GPU):
each rank trains its block of workers on feature shards mapped from the other ranks by
CUDA IPC, gradients are all-reduced; the result must equal the single-process run (ledger
exactly, fp64 losses and weights to summation-order rounding)."""

import os
import pickle
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _setup():
    import paper_2101_07706_b200 as P
    g = P.synth_sbm(P.SbmSpec(n_nodes=900, n_blocks=3, p_in=0.05, p_out=0.005, feature_dim=16,
                              noise_sigma=0.5, seed=2))
    part = P.partition_nodes(g.n_nodes, 4, "random", seed=1)
    return P, g, part


def _train(P, g, part):
    P.set_compute_dtype("float64")
    model = P.init_model([16, 12, 12, 3], 4)
    metrics, ledger = P.train_distributed(g, part, model, P.SamplerConfig(budget=64, skew_constant=8.0,
                                                                          mode="skewed"),
                                          epochs=2, batch_size=48, lr=0.2, mode="skewed", seed=3)
    return [(r.epoch, r.worker, r.loss, r.comm_nodes_epoch) for r in metrics.rows], ledger.counts, model.weights


def _rank_main(rank, world, port, out):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, g, part = _setup()
    res = _train(P, g, part)
    if rank == 0:
        Path(out).write_bytes(pickle.dumps(res))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_training_equals_single_process(tmp_path):
    import torch.multiprocessing as mp
    out = tmp_path / "r0.pkl"
    mp.start_processes(_rank_main, args=(2, 29533, str(out)), nprocs=2, join=True, start_method="spawn")
    rows, ledger, weights = pickle.loads(out.read_bytes())
    P, g, part = _setup()
    rows1, ledger1, weights1 = _train(P, g, part)
    assert np.array_equal(ledger, ledger1)
    assert [r[:2] + r[3:] for r in rows] == [r[:2] + r[3:] for r in rows1]
    np.testing.assert_allclose([r[2] for r in rows], [r[2] for r in rows1], rtol=1e-10)
    for a, b in zip(weights, weights1):
        np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-12)


def _rank_main_det(rank, world, port, out):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, g, part = _setup()
    P.set_compute_dtype("float32")
    model = P.init_model([16, 12, 12, 3], 4)
    metrics, ledger = P.train_distributed(g, part, model, P.SamplerConfig(budget=64, skew_constant=8.0,
                                                                          mode="skewed"),
                                          epochs=2, batch_size=48, lr=0.2, mode="skewed", seed=3,
                                          deterministic=True)
    if rank == 0:
        Path(out).write_bytes(pickle.dumps(([(r.epoch, r.worker, r.loss) for r in metrics.rows],
                                            ledger.counts, model.weights)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_deterministic_mode_is_bit_identical(tmp_path):
    """deterministic=True: per-worker gradients all-gathered and summed in worker order, so
    the 2-process fp32 run equals the single-process one bit for bit (weights and losses)."""
    import torch.multiprocessing as mp
    out = tmp_path / "r0.pkl"
    mp.start_processes(_rank_main_det, args=(2, 29541, str(out)), nprocs=2, join=True, start_method="spawn")
    rows, ledger, weights = pickle.loads(out.read_bytes())
    P, g, part = _setup()
    P.set_compute_dtype("float32")
    model = P.init_model([16, 12, 12, 3], 4)
    metrics, ledger1 = P.train_distributed(g, part, model, P.SamplerConfig(budget=64, skew_constant=8.0,
                                                                           mode="skewed"),
                                           epochs=2, batch_size=48, lr=0.2, mode="skewed", seed=3)
    P.set_compute_dtype("float64")
    assert np.array_equal(ledger, ledger1.counts)
    assert rows == [(r.epoch, r.worker, r.loss) for r in metrics.rows]
    for a, b in zip(weights, model.weights):
        assert np.array_equal(a, b)


def _binary_setup():
    P, g, part = _setup()
    rng = np.random.default_rng(5)
    g.features = (rng.random((g.n_nodes, 256)) < 0.05).astype(np.float64)  # packed on upload
    return P, g, part


def _train_bits(P, g, part):
    P.set_compute_dtype("float64")
    model = P.init_model([256, 12, 12, 3], 4)
    metrics, ledger = P.train_distributed(g, part, model, P.SamplerConfig(budget=64, skew_constant=8.0,
                                                                          mode="skewed"),
                                          epochs=1, batch_size=48, lr=0.2, mode="skewed", seed=3,
                                          deterministic=True)
    return [(r.epoch, r.worker, r.loss) for r in metrics.rows], ledger.counts, model.weights


def _rank_main_bits(rank, world, port, out):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, g, part = _binary_setup()
    res = _train_bits(P, g, part)
    from paper_2101_07706_b200 import _device as D
    res = res + (bool(D.device_graph(g).xbits),)
    if rank == 0:
        Path(out).write_bytes(pickle.dumps(res))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_bit_packed_feature_shards(tmp_path):
    """0/1 features are packed on upload, each rank's shard is uploaded packed and the peer
    shards are read bit-packed through CUDA IPC by the fused layer-0 SpMM; with the ordered
    reduction the 2-process run equals the single-process one bit for bit."""
    import torch.multiprocessing as mp
    out = tmp_path / "r0.pkl"
    mp.start_processes(_rank_main_bits, args=(2, 29547, str(out)), nprocs=2, join=True, start_method="spawn")
    rows, ledger, weights, packed = pickle.loads(out.read_bytes())
    assert packed
    P, g, part = _binary_setup()
    rows1, ledger1, weights1 = _train_bits(P, g, part)
    assert np.array_equal(ledger, ledger1)
    assert rows == rows1
    for a, b in zip(weights, weights1):
        assert np.array_equal(a, b)
