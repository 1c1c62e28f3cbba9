"""Multi-process host logic of the data-parallel path, on CPU with gloo (world size 2).

What crosses ranks in the GPU build: worker-block assignment, the
per-epoch loss/ledger reduction, the gradient all-reduce of per-rank worker-ordered sums,
and the node -> (rank, row) feature-shard map that the NVLink gather reads.  The same
functions run here on CPU tensors.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2101_07706_b200.training import (assign_workers, feature_shard_map, reduce_epoch_stats,
                                            worker_ranks)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k, L, epochs = 8, 5, 2
        active = [0, 1, 2, 4, 5, 6, 7]          # worker 3 has no training nodes
        mine = assign_workers(active, rank, world)
        r = np.random.default_rng(123)
        grads = r.normal(size=(k, 64))           # every rank can regenerate every worker's
        losses = r.uniform(0.5, 2.0, size=(k, 3))
        ledger_all = r.integers(0, 500, size=(epochs, k, L))
        # gradient all-reduce of per-rank, worker-ordered partial sums
        g = torch.zeros(64, dtype=torch.float64)
        for w in mine:
            g += torch.as_tensor(grads[w])
        dist.all_reduce(g)
        # epoch statistics
        loss_sum = np.zeros(k)
        loss_cnt = np.zeros(k, dtype=np.int64)
        for w in mine:
            for it in range(3):
                loss_sum[w] += losses[w, it]
                loss_cnt[w] += 1
        led = torch.zeros((k, L), dtype=torch.int64)
        for w in mine:
            led[w] = torch.as_tensor(ledger_all[0, w])
        ls, lc, led = reduce_epoch_stats(dist, loss_sum, loss_cnt, led)
        q.put((rank, mine, g.numpy(), ls, lc, led.numpy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_reductions_match_single_process():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda x: x[0])
    k, L = 8, 5
    active = [0, 1, 2, 4, 5, 6, 7]
    r = np.random.default_rng(123)
    grads = r.normal(size=(k, 64))
    losses = r.uniform(0.5, 2.0, size=(k, 3))
    ledger_all = r.integers(0, 500, size=(2, k, L))
    # worker blocks are contiguous, disjoint, and cover the active list in order
    assert out[0][1] + out[1][1] == active
    ref_g = sum(grads[w] for w in active)
    ref_ls = np.zeros(k)
    for w in active:
        for it in range(3):
            ref_ls[w] += losses[w, it]
    for rank, mine, g, ls, lc, led in out:
        np.testing.assert_allclose(g, ref_g, rtol=1e-12)
        np.testing.assert_array_equal(ls, ref_ls)          # single contributor per entry: exact
        np.testing.assert_array_equal(lc, [3 if w in active else 0 for w in range(k)])
        exp_led = np.zeros((k, L), dtype=np.int64)
        exp_led[active] = ledger_all[0, active]
        np.testing.assert_array_equal(led, exp_led)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_assign_workers_partitions_active_list(world):
    for active in ([0, 1, 2, 3, 4, 5, 6, 7], [1, 3, 4], list(range(13)), [5]):
        blocks = [assign_workers(active, r, world) for r in range(world)]
        assert sum(blocks, []) == list(active)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_feature_shard_map_round_trip(world):
    r = np.random.default_rng(world)
    k, n = 8, 5000
    owner = r.integers(0, k, size=n)
    active = [w for w in range(k) if w != 2]
    wr = worker_ranks(k, active, world)
    node_rank, node_row, rows = feature_shard_map(owner, wr, world)
    assert sum(len(x) for x in rows) == n
    for node in r.choice(n, 200, replace=False):
        rk, rw = node_rank[node], node_row[node]
        assert rows[rk][rw] == node
        assert rk == wr[owner[node]]
    for x in rows:
        assert np.all(np.diff(x) > 0)
