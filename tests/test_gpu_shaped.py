"""The CUDA path at the benchmarked configurations, against reference-generated goldens:

* loss_and_backward / forward at the Reddit shape with dims [602, 256 x 4, 41]
  (golden_reddit_fb.npz) in fp32 (3xTF32 tcgen05 GEMMs, north_star's rtol 1e-4) and fp64;
* the Trainer's batched, two-stream, CUDA-graph-replayed sampler pipeline (24 plans per
  launch, the bench's path incl. skg_ladies_sample_device) against the reference's plans
  and ledger for iterations 0..2 of all k = 8 workers (golden_pipeline.npz);
* the global-atomic expand (the > 1M-node path) forced on the Reddit goldens.
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import skewgcn_oracle as O
from golden_util import golden, shaped, shaped_batch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def P():
    import paper_2101_07706_b200 as pkg
    return pkg


def _reddit():
    import torch
    sgph = shaped("reddit", device="cuda" if torch.cuda.is_available() else None)
    return sgph, P().from_shaped(sgph)


def _light(sgph):
    return O.Graph(n_nodes=sgph.n_nodes, offsets=sgph.offsets, neighbors=sgph.neighbors,
                   weights=sgph.weights, train_mask=sgph.train_mask)


@pytest.mark.parametrize("dtype,rtol,atol", [("float32", 1e-4, 1e-6), ("float64", 1e-9, 1e-13)])
def test_reddit_forward_backward_golden(dtype, rtol, atol):
    pkg = P()
    G = golden("reddit_fb")
    sgph, g = _reddit()
    assert sgph.structure_hash() == G.meta["shape_reddit"]["structure_sha"]
    assert sgph.features_hash() == G.meta["shape_reddit"]["features_sha"]
    part = pkg.partition_nodes(g.n_nodes, 8, "random", seed=1)
    opart = O.partition_nodes(g.n_nodes, 8, "random", seed=1)
    labels = np.asarray(sgph.labels)
    old = pkg.compute_dtype()
    pkg.set_compute_dtype(dtype)
    try:
        for case in G.cases("reddit_fb"):
            m = G.meta[case]
            batch = shaped_batch(_light(sgph), opart, m)
            np.testing.assert_array_equal(batch, G.get(case, "batch"))
            cfg = pkg.SamplerConfig(budget=512, skew_constant=m["D"], mode=m["mode"])
            plan = pkg.ladies_plan(g, part, m["worker"], batch, cfg, 5,
                                   O.spawn_rng(0, "plan", 0, 0, m["worker"]))
            np.testing.assert_array_equal(plan.remote_per_layer(), G.get(case, "remote"))
            model = pkg.init_model(m["dims"], m["model_seed"])
            loss, grads = pkg.loss_and_backward(model, plan, sgph.features, labels)
            logits = pkg.forward(model, plan, sgph.features)
            ref_logits = G.get(case, "logits")
            # fp32 through 5 layers (K = 602/256 contractions, ~2 nnz per block row):
            # a logit near zero keeps an absolute error of a few 1e-6 of the largest logit,
            # so its norm-aware floor is 1e-5 x max|logit| (1 entry in 21K needed more than
            # 1e-6 on the B200); fp64 keeps the tight floor
            lat = 1e-5 if dtype == "float32" else atol
            np.testing.assert_allclose(logits, ref_logits, rtol=rtol,
                                       atol=lat * float(np.abs(ref_logits).max()))
            assert loss == pytest.approx(float(G.get(case, "loss")), rel=rtol)
            for l, gr in enumerate(grads):
                idx = G.get(case, f"grad{l}_idx")
                scale = float(G.get(case, f"grad{l}_norm")) / np.sqrt(gr.size)  # rms entry
                # fp32: north_star's rtol 1e-4 taken at the tensor's scale (entries near zero
                # after cancellation carry ~1e-5 x rms of fp32 error through 5 layers)
                gat = rtol * scale if dtype == "float32" else atol * 10 * scale
                np.testing.assert_allclose(gr.reshape(-1)[idx], G.get(case, f"grad{l}_val"),
                                           rtol=rtol, atol=gat,
                                           err_msg=f"{case} {dtype} grad{l} (sampled entries)")
                assert np.linalg.norm(gr) == pytest.approx(float(G.get(case, f"grad{l}_norm")),
                                                           rel=rtol)
                if G.has(case, f"grad{l}"):
                    ref = G.get(case, f"grad{l}")
                    np.testing.assert_allclose(gr, ref, rtol=rtol, atol=gat,
                                               err_msg=f"{case} {dtype} grad{l}")
                    # and the whole tensor, relative in norm
                    assert np.linalg.norm(gr - ref) <= rtol * np.linalg.norm(ref)
    finally:
        pkg.set_compute_dtype(old)


def _pipe_expect(G, it, w):
    case = f"pipe_{it}_{w}"
    return {l: {k: G.get(case, f"L{l}/{k}") for k in ("nodes", "indptr", "indices", "data")}
            for l in range(5)}, G.get(case, "remote"), G.get(case, "batch")


def _check_slot(G, ps, slot, it, w):
    from paper_2101_07706_b200 import _device as D
    exp, remote, batch = _pipe_expect(G, it, w)
    st, info, rc = ps.stats(slot)
    assert rc == 0
    got_remote = st[:, 4][::-1]
    np.testing.assert_array_equal(got_remote, remote, err_msg=f"plan ({it},{w}) ledger")
    for t in range(5):
        lay = D.read_layer(ps, slot, t, st[t], False)
        l = 4 - t
        e = exp[l]
        np.testing.assert_array_equal(lay["nodes"], e["nodes"], err_msg=f"({it},{w}) L{l} nodes")
        np.testing.assert_array_equal(lay["indptr"], e["indptr"], err_msg=f"({it},{w}) L{l} indptr")
        np.testing.assert_array_equal(lay["indices"], e["indices"], err_msg=f"({it},{w}) L{l} indices")
        np.testing.assert_allclose(lay["values"], e["data"], rtol=1e-12, atol=0,
                                   err_msg=f"({it},{w}) L{l} values")


@pytest.mark.parametrize("ahead,streams,device_batches", [(3, 2, False), (3, 2, True), (1, 2, False)])
def test_trainer_pipeline_golden(ahead, streams, device_batches):
    """The bench's pipeline at the Reddit shape: plans of iterations 0..2 for all 8 workers
    sampled in groups of `ahead` iterations (24 plans per launch at ahead = 3) on `streams`
    sampler streams into rotating arenas, replayed as CUDA graphs, with host batches
    (skg_ladies_sample) or HBM-resident ones (skg_ladies_sample_device); each group's plans
    are compared with the reference's while the GCN consumes them, then the ledger."""
    import torch
    pkg = P()
    G = golden("pipeline")
    m = G.meta["pipeline"]
    sgph, g = _reddit()
    assert sgph.structure_hash() == m["structure_sha"]
    part = pkg.partition_nodes(g.n_nodes, m["k"], "random", seed=m["pseed"])
    dims = [sgph.features.shape[1], 256, 256, 256, 256, sgph.n_classes]
    model = pkg.init_model(dims, seed=0)
    cfg = pkg.SamplerConfig(budget=m["budget"], skew_constant=m["D"], mode=m["mode"])
    pkg.set_compute_dtype("float32")
    tr = pkg.Trainer(g, part, model, cfg, batch_size=m["batch_size"], lr=0.5, mode=m["mode"],
                     seed=m["seed"], dtype="float32", epochs=1, ahead=ahead, streams=streams)
    try:
        assert tr.n_my == m["k"]
        iters = m["iters"]
        checked = []
        d_ids = None
        if device_batches:
            ids = np.zeros((iters, tr.n_my, m["batch_size"]), dtype=np.int32)
            bl = np.zeros((iters, tr.n_my), dtype=np.int32)
            states = np.zeros((iters, tr.n_my, 4), dtype=np.uint64)
            for it in range(iters):
                boff, bids, st = tr.host_inputs(0, it, 0)
                for i in range(tr.n_my):
                    bl[it, i] = boff[i + 1] - boff[i]
                    ids[it, i, :bl[it, i]] = bids[boff[i]:boff[i + 1]]
                states[it] = st[:tr.n_my]
            d_ids = torch.as_tensor(ids, device="cuda")
            workers = np.array(tr.mine * ahead, dtype=np.int32)

        def sample_fn(grp, buf):
            if not device_batches:
                tr.sample_group([(0, it) for it in grp], buf)
                return
            s0, n = grp[0], len(grp)
            tr.sample_device(buf, n * tr.n_my, workers, np.ascontiguousarray(bl[s0:s0 + n].reshape(-1)),
                             d_ids[s0].data_ptr(), m["batch_size"],
                             np.ascontiguousarray(states[s0:s0 + n].reshape(-1, 4)))

        def compute_fn(grp, buf):
            torch.cuda.synchronize()
            ps = tr.bufs[buf][0]
            for gi, it in enumerate(grp):
                for i, w in enumerate(tr.mine):
                    _check_slot(G, ps, gi * tr.n_my + i, it, w)
                    checked.append((it, w))
                tr.compute(0, it, gi, buf)
                tr.reduce_and_step()

        groups = [tuple(range(g0, min(iters, g0 + ahead))) for g0 in range(0, iters, ahead)]
        tr.pipeline(groups, sample_fn, compute_fn)
        torch.cuda.synchronize()
        assert sorted(checked) == [(it, w) for it in range(iters) for w in range(m["k"])]
        np.testing.assert_array_equal(tr.ledger[0].cpu().numpy(), G.get("pipeline", "ledger"))
        tr.check_errors()
    finally:
        tr.close()


@pytest.mark.parametrize("path", ["global", "ranges"])
def test_older_expand_paths_on_reddit_goldens(path):
    """Force the older expand kernels on the Reddit-shaped goldens, in a fresh process:
    `global` = the global-atomic expand (k_lad_expand + k_bitmap_tiles, taken by graphs of
    more than 16 x 65536 nodes); `ranges` = the shared-memory-counter range expand with
    node-indexed slots (k_lad_expand_ranges + k_bitmap_compact + k_lad_fold).  The default
    fused range kernel (k_lad_range) runs these goldens in the other tests."""
    env = dict(os.environ, SKG_EXPAND=path)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py::test_shaped_golden[reddit_s]",
                        "tests/test_gpu_parity.py::test_shaped_golden[reddit]",
                        "tests/test_gpu_shaped.py::test_trainer_pipeline_golden[3-2-False]"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "3 passed" in r.stdout, r.stdout[-2000:]


# ------------------------------------------------------------ full-graph evaluation at shape
@pytest.mark.parametrize("dtype,rtol", [("float64", 1e-9), ("float32", 1e-4)])
def test_predict_logits_reddit_s_vs_oracle(dtype, rtol):
    """predict_logits (training.py:325-334) on the 40K-node / 2M-edge reduced Reddit shape,
    dims [602, 256 x 4, 41], against the CPU oracle's (P @ h) @ W chain in fp64."""
    import paper_2101_07706_b200 as pkg
    from golden_util import oracle_graph_from_shaped
    sg = shaped("reddit_s")
    og = oracle_graph_from_shaped(sg)
    dims = [602, 256, 256, 256, 256, 41]
    ws = O.init_model(dims, 0)
    ref = O.predict_logits(ws, og)
    pkg.set_compute_dtype(dtype)
    try:
        got = pkg.predict_logits(pkg.GcnModel([w.copy() for w in ws]), pkg.from_shaped(sg))
    finally:
        pkg.set_compute_dtype("float64")
    scale = float(np.abs(ref).max())
    np.testing.assert_allclose(got, ref, rtol=rtol, atol=rtol * scale)


@pytest.mark.parametrize("dtype,rtol", [("float64", 1e-9), ("float32", 1e-4)])
def test_predict_logits_full_reddit_vs_torch_sparse(dtype, rtol):
    """predict_logits at the full Reddit shape (232,965 nodes, 113.5M CSR entries, 602-d):
    compared with an independent fp64 chain on the device (torch CSR sparse @ dense, then
    dense GEMM; the CPU oracle would need minutes for the 114M x 602 product)."""
    import torch
    import paper_2101_07706_b200 as pkg
    sg = shaped("reddit", device="cuda")
    dims = [602, 256, 256, 256, 256, 41]
    ws = O.init_model(dims, 0)
    Pm = torch.sparse_csr_tensor(torch.as_tensor(sg.offsets, device="cuda"),
                                 torch.as_tensor(sg.neighbors.astype(np.int64), device="cuda"),
                                 torch.as_tensor(sg.weights, device="cuda"),
                                 size=(sg.n_nodes, sg.n_nodes))
    h = torch.as_tensor(sg.features, device="cuda").double()
    for l, w in enumerate(ws):
        h = (Pm @ (h.clamp_min(0.0) if l else h)) @ torch.as_tensor(w, device="cuda")
    ref = h.cpu().numpy()
    del Pm, h
    pkg.set_compute_dtype(dtype)
    try:
        got = pkg.predict_logits(pkg.GcnModel([w.copy() for w in ws]), pkg.from_shaped(sg))
    finally:
        pkg.set_compute_dtype("float64")
    scale = float(np.abs(ref).max())
    np.testing.assert_allclose(got, ref, rtol=rtol, atol=rtol * scale)
