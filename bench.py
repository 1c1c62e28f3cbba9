"""Benchmark: LADIES 5-layer GCN training iterations/sec on the Reddit-shaped graph.

Workload (BASELINE.json configs[1]): Reddit-shaped synthetic graph (232,965 nodes,
~114M CSR entries incl. self-loops, 602-d fp32 features, 41 classes), random partition
into k = 8 workers (seed 1), LADIES skewed D = 8, batch 512, budget 512 per layer,
5 layers hidden 256, SGD.  One step = one data-parallel iteration of
train_distributed (training.py:483-506): every worker samples its plan, runs
forward/backward, gradients are averaged over workers (NCCL all-reduce across GPUs)
and the SGD step is applied.  The k = 8 workers are spread over the N GPUs (8/N each),
so the total work per step is fixed: "scaling": "strong".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU oracle port (oracle/skewgcn_oracle.py, a restatement of
the reference's numpy/scipy path) on this host's cores, one worker-iteration per step.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LADIES 5-layer GCN iters/sec at 1/2/4/8 B200; remote nodes fetched/iter"
DIMS_HIDDEN = 256
N_LAYERS = 5
PLANS_PER_LAUNCH = 40  # default sampler look-ahead, in plans (all workers of T iterations)


def parse():
    return parse_args(sys.argv[1:])


def parse_args(argv):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shape", default="reddit")
    ap.add_argument("--sampler", default="auto", choices=["auto", "ladies", "saint"],
                    help="auto: GraphSAINT for the Amazon shape (configs[3]), LADIES otherwise")
    ap.add_argument("--hidden", type=int, default=0, help="0: 512 for Amazon, else 256")
    ap.add_argument("--subgraph", type=int, default=4500, help="GraphSAINT subgraph size")
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--mode", default="skewed")
    ap.add_argument("--D", type=float, default=8.0)
    ap.add_argument("--batch", type=int, default=512)
    ap.add_argument("--budget", type=int, default=512)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--lr", type=float, default=0.0, help="0: 0.5 (LADIES), 0.05 (GraphSAINT)")
    ap.add_argument("--cpu-sample-s", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ahead", type=int, default=0,
                    help="iterations of plans per sampler launch (0: ceil(40 / workers per rank))")
    ap.add_argument("--streams", type=int, default=2, help="sampler streams (groups in flight)")
    a = ap.parse_args(argv)
    if a.sampler == "auto":
        a.sampler = "saint" if a.shape.startswith("amazon") else "ladies"
    if a.lr <= 0:  # GraphSAINT's 1/p-weighted 4500-node blocks diverge at 0.5 with hidden 512
        a.lr = 0.05 if a.sampler == "saint" else 0.5
    if a.hidden <= 0:
        a.hidden = 512 if a.shape.startswith(("amazon", "youtube")) else DIMS_HIDDEN
    return a


def workload_name(args):
    if args.shape.startswith("youtube"):
        return (f"{args.shape}-shaped LADIES {args.mode} D={args.D:g}, k={args.workers} workers, "
                f"batch {args.batch}, budget {args.budget}, {N_LAYERS} layers hidden {args.hidden}, "
                "multi-label BCE pos_weight 50")
    if args.sampler == "saint":
        return (f"{args.shape}-shaped GraphSAINT {args.mode} D={args.D:g}, k={args.workers} workers, "
                f"subgraph {args.subgraph}, {N_LAYERS} layers hidden {args.hidden}")
    return (f"{args.shape}-shaped LADIES {args.mode} D={args.D:g}, k={args.workers} workers, "
            f"batch {args.batch}, budget {args.budget}, {N_LAYERS} layers hidden {args.hidden}")


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock / throttle reasons polled in-process through NVML every ~2 ms while the
    timed region runs (nvidia-smi's start-up is longer than a sub-second timed region);
    falls back to an `nvidia-smi -lms` child process when NVML is unavailable."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []   # (sm_mhz, reasons bitmask)
        self.max_mhz = None
        self._stop = threading.Event()
        self.nv = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            dev = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(self.index)).split(",")[self.index]) \
                if os.environ.get("CUDA_VISIBLE_DEVICES", "").replace(",", "").isdigit() else self.index
            self.h = nv.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.nv = nv
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
                self.samples.append((mhz, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], self.max_mhz, set()
        if self.nv is not None:
            nv = self.nv
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            for mhz, rs in self.samples:
                sm.append(mhz)
                for nm, b in bits.items():
                    if rs & b:
                        reasons.add(nm)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.nv is not None else "nvidia-smi"}


# ---------------------------------------------------------------------------- setup
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 and relay their output."""
    import socket
    if os.environ.get("SKG_DIST_BACKEND", "nccl") == "nccl" and args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, "
                             f"this node has {have} (SKG_DIST_BACKEND=gloo shares GPUs for "
                             "functional runs)\n")
            return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def shape_info(shape):
    from importlib.util import module_from_spec, spec_from_file_location
    # synth.py by path: the reference arm must not import the package (which maps libskg)
    if "skg_synth" in sys.modules:
        return sys.modules["skg_synth"]
    spec = spec_from_file_location("skg_synth", ROOT / "paper_2101_07706_b200" / "synth.py")
    mod = module_from_spec(spec)
    sys.modules["skg_synth"] = mod  # dataclasses resolve their module through sys.modules
    spec.loader.exec_module(mod)
    return mod


def bench_config(args, n_nodes, nnz, feat_dim):
    """The workload description both arms print (identical dicts: same_config)."""
    l2_mb = 126
    cols_mb = nnz * 4 / 1e6
    packed = args.shape.startswith("youtube")  # build_workload stores these rows bit-packed
    feat_mb = n_nodes * (((feat_dim + 31) // 32) * 4 if packed else feat_dim * 4) / 1e6
    feat = "bit-packed features" if packed else "fp32 features"
    touch = ("every plan touches ~2/3 of the nodes" if args.shape.startswith("reddit")
             else "each step samples fresh random batches")
    return {"workload": workload_name(args), "n_nodes": int(n_nodes), "nnz": int(nnz),
            "feature_dim": int(feat_dim), "workers": args.workers,
            "l2": (f"inputs > L2: {cols_mb:.0f} MB of CSR columns and {feat_mb:.0f} MB of "
                   f"{feat} against a {l2_mb} MB L2, {touch}; no flush between steps")}


def build_workload(args, device):
    from paper_2101_07706_b200.synth import make_shaped_graph
    t0 = time.time()
    # YouTube's 2048-d multi-hot rows are generated and stored bit-packed (32 per word)
    sg = make_shaped_graph(args.shape, seed=0, device=device, packed=args.shape.startswith("youtube"))
    return sg, time.time() - t0


def plan_bytes_8d(st_rows, budget, saint=False):
    """SURVEY §8(d), verbatim: LADIES, per sampled layer,
    8*E_l + 12*|S_{l+1}| + 25*N_l + 8*B + 12*nnz_l + 12*|S_l|;  GraphSAINT, per plan,
    17*N + 8*B + 8*E_sub + 12*|sub| + 12*nnz.  (Saturated layers draw nothing: no 8*B.)
    stats columns: 0 n_upper, 1 n_cand, 2 n_nodes, 3 nnz, 5 has_dist, 9 n_pairs."""
    if saint:
        r = st_rows[0]
        n_sub, nnz = int(r[2]), int(r[3])
        # E_sub: adjacency entries the induced-block filter reads (the sub rows' degrees);
        # the sampler stores nnz of sub x sub, E_sub = the pairs it scanned (n_pairs)
        e_sub = int(r[9]) if int(r[9]) else nnz
        return 17 * int(r[1]) + 8 * budget + 8 * e_sub + 12 * n_sub + 12 * nnz
    total = 0
    for r in st_rows:
        n_upper, n_cand, n_nodes, nnz = (int(x) for x in r[:4])
        draws = 8 * budget if int(r[5]) else 0
        total += 8 * int(r[9]) + 12 * n_upper + 25 * n_cand + draws + 12 * nnz + 12 * n_nodes
    return total


# per-kernel shares of the §8(d) LADIES layer formula (they sum to it): the expansion reads
# the upper rows' columns and degrees; the compaction the owner byte; the fold writes the
# fp64 norm, the pairwise / probability pass reads it; the exact cumsum writes the fp64
# cdf; the draws read B uniforms and emit ids + p; the block pass writes col + value
def kernel_bytes_8d(stats, budget):
    E = sum(int(r[9]) for st in stats for r in st)
    U = sum(int(r[0]) for st in stats for r in st)
    N = sum(int(r[1]) for st in stats for r in st)
    S = sum(int(r[2]) for st in stats for r in st)
    Z = sum(int(r[3]) for st in stats for r in st)
    B = sum(budget for st in stats for r in st if int(r[5]))
    return {"k_lad_expand_ranges": 8 * E + 12 * U, "k_lad_expand": 8 * E + 12 * U,
            # the fused range kernel does the expansion, compaction and fold shares
            "k_lad_range": 8 * E + 12 * U + 9 * N,
            "k_bitmap_compact": 1 * N, "k_lad_fold": 8 * N, "k_pw_leaves": 8 * N,
            "k_cs_maps": 8 * N, "k_draw_dedup": 8 * B + 12 * S, "k_lad_finish": 12 * Z}


# ---------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    world, rank, local = dist_setup(args)
    # one process per GPU; more ranks than GPUs (functional checks on a one-GPU box) share
    # devices round-robin and must use SKG_DIST_BACKEND=gloo (NCCL needs distinct GPUs)
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    local = dev
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("SKG_DIST_BACKEND", "nccl")
        if backend == "nccl":
            # communicator lines (ranks, NVLink / NVLS channels) in the run log
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    import paper_2101_07706_b200 as P
    from paper_2101_07706_b200._native import lib

    sg, t_gen = build_workload(args, f"cuda:{local}")
    g = P.from_shaped(sg)
    k = args.workers
    part = P.partition_nodes(sg.n_nodes, k, "random", seed=1)
    dims = [sg.features.shape[1]] + [args.hidden] * (N_LAYERS - 1) + [sg.n_classes]
    model = P.init_model(dims, seed=0)
    saint = args.sampler == "saint"
    cfg = P.SamplerConfig(budget=args.subgraph if saint else args.budget, skew_constant=args.D,
                          mode=args.mode)
    P.set_compute_dtype(args.dtype)
    # the Trainer's GCN runs on the caller's stream: a high-priority one (the sampler streams
    # run at the lowest priority), as train_distributed does
    torch.cuda.set_stream(torch.cuda.Stream(priority=int(os.environ.get("SKG_MAIN_PRIO", "-1"))))
    # plans per sampler launch stay ~40 whatever the rank count (k = 8 workers per step,
    # spread over the ranks): look-ahead T = ceil(40 / workers on this rank).  Measured on
    # one B200 (Reddit LADIES): T = 3 / 4 / 5 / 6 -> 2030 / 2077 / 2095 / 2051 it/s
    n_my_est = max(1, len(P.training.assign_workers(list(range(k)), rank, world)))
    T = args.ahead if args.ahead > 0 else max(1, -(-PLANS_PER_LAUNCH // n_my_est))
    tr = P.Trainer(g, part, model, cfg, batch_size=args.batch, lr=args.lr, mode=args.mode,
                   seed=0, dtype=args.dtype, epochs=1, ahead=T, streams=args.streams,
                   sampler=args.sampler, subgraph_size=args.subgraph if saint else None)
    stream = torch.cuda.current_stream()
    n_my = tr.n_my
    S = tr.n_streams
    K = max(args.steps, 1)
    W = max(args.warmup, 0)
    TAIL = S * T  # plans sampled ahead at the end of a timed region (the look-ahead)
    per = tr.per_epoch

    # ---- inputs resident in HBM: batch ids + plan states of every step, derived up front
    total_steps = W + K + TAIL
    bl = np.zeros((total_steps, n_my), dtype=np.int32)
    states = np.zeros((total_steps, n_my, 4), dtype=np.uint64)
    ids = np.zeros((total_steps, n_my, args.batch), dtype=np.int32)
    for st_i in range(total_steps):
        boff, bids, st = tr.host_inputs(st_i // per, st_i % per, 0)
        if not saint:  # GraphSAINT plans draw from the training set: rng states only
            for i in range(n_my):
                n_i = boff[i + 1] - boff[i]
                bl[st_i, i] = n_i
                ids[st_i, i, :n_i] = bids[boff[i]:boff[i + 1]]
        states[st_i] = st[:n_my]
    d_ids = torch.as_tensor(ids, device="cuda")
    workers = np.array(tr.mine * T, dtype=np.int32)

    def sample_resident(s0, n, buf):
        if saint:
            tr._states[:n * n_my] = states[s0:s0 + n].reshape(-1, 4)
            tr.sample(n * n_my, buf)
            return
        tr.sample_device(buf, n * n_my, workers, np.ascontiguousarray(bl[s0:s0 + n].reshape(-1)),
                         d_ids[s0].data_ptr(), args.batch,
                         np.ascontiguousarray(states[s0:s0 + n].reshape(-1, 4)))

    def groups_of(s0, count):
        return [(g0, min(T, s0 + count - g0)) for g0 in range(s0, s0 + count, T)]

    no_gcn = bool(os.environ.get("SKG_BENCH_SAMPLER_ONLY"))  # diagnostic: pipeline minus GCN

    def compute_group(grp, b):
        g0, n = grp
        for i in range(n):
            if no_gcn:
                continue
            tr.compute(0, (g0 + i) % per, i, b)
            tr.reduce_and_step()

    def steps_resident(s0, count, ahead_count):
        # the Trainer's pipeline: groups sampled ahead on the sampler streams into rotating
        # plan arenas while the GCN consumes them in order on the main stream; the first
        # groups of the next call are sampled ahead too (steady state across calls)
        tr.pipeline(groups_of(s0, count), lambda grp, b: sample_resident(grp[0], grp[1], b),
                    compute_group, next_groups=groups_of(s0 + count, ahead_count))

    def steps_serial(s0, count):
        # the same steps with the stages serialised (a group's sampling, then its GCN steps,
        # nothing overlapped): per-kernel times as a serialised profiler sees them
        tr.drop_pending()
        torch.cuda.synchronize()
        for g0, n in groups_of(s0, count):
            sample_resident(g0, n, 0)
            tr.wait_sampled(0)
            for i in range(n):
                tr.compute(0, (g0 + i) % per, i, 0)
                tr.reduce_and_step()
            tr.release_buf(0)
            torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- every CUDA graph the run replays (each arena x full / partial group sizes, GCN
    # steps at each group offset) is captured and instantiated here, without running it,
    # so the warm-up is exactly W steps and no capture lands in a timed region
    prepare_graphs(tr, lib, sample_resident, T, n_my, [T, W % T, K % T, (W + K) % T])

    # ---- warm-up: W steps; the look-ahead of the timed region is sampled at its end
    steps_resident(0, W, K)
    barrier()
    launches0 = P.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fr_trace = os.environ.get("SKG_FR_TRACE")  # diagnostic: range-expand CTA timeline
    if fr_trace:
        lib.skg_debug_fr_trace(1 + int(os.environ.get("SKG_FR_TRACE_THREAD", "0")), None)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for sd in tr.sides:  # the sampler streams start inside the timed region
            sd.wait_event(ev0)
        h0 = time.perf_counter()
        if os.environ.get("SKG_BENCH_PROFILE"):  # host-side profile of the timed loop
            import cProfile
            import pstats
            prof = cProfile.Profile()
            prof.runcall(steps_resident, W, K, TAIL)
            pstats.Stats(prof, stream=sys.stderr).sort_stats("tottime").print_stats(25)
        else:
            steps_resident(W, K, TAIL)
        host_ms = (time.perf_counter() - h0) * 1e3  # enqueue time (the loop never syncs)
        for sd in tr.sides:  # the region ends when the look-ahead sampling ends too
            stream.wait_stream(sd)
        ev1.record(stream)
        barrier()
    launches = P.kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1)
    if fr_trace:
        buf = (C.c_ulonglong * (8 * 32 * 11))()
        lib.skg_debug_fr_trace(0, buf)
        with open(fr_trace, "w") as fh:
            json.dump(list(buf), fh)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    tr.check_errors()
    ms_per_step = ms / K

    # ---- ledger, plan statistics and the per-stage split (separate instrumented pass)
    ledger = tr.ledger[0].clone()
    if dist is not None:
        dist.all_reduce(ledger)
    steps_done = W + K
    remote_per_iter = float(ledger.sum().item()) / steps_done
    torch.cuda.synchronize()
    tr.drop_pending()
    steps_serial(W, min(T, K))  # one full group in arena 0: its plans' statistics
    stats = [tr.bufs[0][0].stats(i)[0] for i in range(n_my * min(T, K))]
    n_it = min(T, K)
    # GraphSAINT plans record their one subgraph (shared by every GCN layer) as layer 0
    in_layer = 0 if saint else N_LAYERS - 1
    s0_rows = sum(int(st[in_layer, 2]) for st in stats) / n_it          # |S_0| per iteration
    s0_remote = sum(int(st[in_layer, 4]) for st in stats) / n_it        # remote rows moved
    sampled_nodes = (sum(int(st[0, 2]) for st in stats) if saint
                     else sum(int(st[:, 2].sum()) for st in stats)) / n_it
    budget = args.subgraph if saint else args.budget
    alg_bytes = sum(plan_bytes_8d(st, budget, saint) for st in stats)  # n_it iterations' plans
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    samp_ms, comp_ms = [], []
    for rep in range(3):  # stages run back to back here (no overlap) to time each alone
        s0 = W + (rep * n_it) % max(1, K - n_it + 1)
        torch.cuda.synchronize()
        ev[0].record(tr.side)
        sample_resident(s0, n_it, 0)
        ev[1].record(tr.side)
        tr.wait_sampled(0)
        torch.cuda.synchronize()
        ev[2].record(stream)
        ev[3].record(stream)
        for gi in range(n_it):
            tr.compute(0, (s0 + gi) % per, gi, 0)
            tr.reduce_and_step()
        ev[4].record(stream)
        tr.release_buf(0)
        torch.cuda.synchronize()
        samp_ms.append(ev[0].elapsed_time(ev[1]))
        comp_ms.append(ev[3].elapsed_time(ev[4]) / n_it)
    samp = float(np.median(samp_ms))  # one launch sequence of n_it iterations' plans
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    achieved = alg_bytes / (samp * 1e-3) / 1e9

    # ---- per-kernel live timing: CUDA events around every launch of every kernel (on its
    # stream) over the K timed steps replayed with the stages serialised
    steps_serial(W, K)  # eager launches: first-use work before the profiled pass
    kern, _ = kernel_table(lib, steps_serial, W, K, stats, tr, T, peaks, saint, budget)
    top = max(kern, key=lambda r: r["total_ms"])
    dominant = top["kernel"]
    if top["frac"] is None:  # no algorithmic model: report the largest modelled kernel
        top = max((r for r in kern if r["frac"] is not None), key=lambda r: r["total_ms"])
    # the layer-0 row gather (local or NVLink peer rows) is fused into the first SpMM
    gather = [r for r in kern if r["kernel"].startswith(("k_gather_b", "k_spmm_in_b"))]

    # ---- all-reduce of the gradient (NCCL across ranks), timed alone
    ar = None
    if dist is not None:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for _ in range(3):
            dist.all_reduce(tr.gflat)
        torch.cuda.synchronize()
        evs[0].record(stream)
        for _ in range(20):
            dist.all_reduce(tr.gflat)
        evs[1].record(stream)
        torch.cuda.synchronize()
        ar_ms = evs[0].elapsed_time(evs[1]) / 20
        ar_bytes = tr.gflat.numel() * tr.gflat.element_size()
        ar = {"bytes": int(ar_bytes), "ms_per_step": round(ar_ms, 4),
              "bus_gbs": round(ar_bytes * 2 * (world - 1) / world / (ar_ms * 1e-3) / 1e9, 2),
              "backend": dist.get_backend()}

    # ---- e2e through the public API (Trainer.run): host-derived inputs, H2D every group,
    # every step's loss read back to the host; steady state like the device region (the
    # warm-up samples the region's first groups, the region samples the next call's)
    tr.drop_pending()
    barrier()
    h2d = [0]
    LAG = max(2, 3 * T)
    RING = LAG + 2
    ring = [torch.empty(n_my, dtype=torch.float64, pin_memory=True) for _ in range(RING)]
    ring_ev = [torch.cuda.Event() for _ in range(RING)]
    pending, host_losses = [], []
    counting = [False]

    def read_loss(e, it):
        # each step's loss is copied to pinned host memory behind its GCN on the main stream
        # and read by the host LAG steps later (the host stays as far ahead as the sampler
        # look-ahead); every loss of the region is read inside it
        if counting[0]:
            h2d[0] += int(tr._boff[n_my]) * 4 + n_my * 32
        i = len(host_losses) + len(pending)
        ring[i % RING].copy_(tr.losses[it % per], non_blocking=True)
        ring_ev[i % RING].record(stream)
        pending.append(i)
        while len(pending) > LAG:
            j = pending.pop(0)
            ring_ev[j % RING].synchronize()
            host_losses.append(float(ring[j % RING].sum()))

    def drain():
        while pending:
            j = pending.pop(0)
            ring_ev[j % RING].synchronize()
            host_losses.append(float(ring[j % RING].sum()))

    pairs = [(s_ // per, s_ % per) for s_ in range(W + K + TAIL)]
    tr.run(pairs[:W], on_iteration=read_loss, next_pairs=pairs[W:W + K])
    drain()
    barrier()
    n_before = len(host_losses)
    counting[0] = True
    t_e2e0 = time.perf_counter()
    tr.run(pairs[W:W + K], on_iteration=read_loss, next_pairs=pairs[W + K:])
    drain()
    torch.cuda.synchronize()  # includes the look-ahead sampling of the next call's groups
    barrier()
    e2e_ms = (time.perf_counter() - t_e2e0) * 1e3
    counting[0] = False
    assert len(host_losses) - n_before == K, "e2e: step losses not all read"
    tr.check_errors()
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    out = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1 and tr.multilabel:
            cpu = {"value": None, "unavailable": "the reference has no multi-label (BCE) loss; "
                                                 "no CPU implementation to time"}
        elif not args.no_cpu_baseline and world == 1:
            norms = None
            if saint and args.mode != "local":  # bit-exact with the oracle's (parity tests)
                norms = P.train_column_norms(g, np.flatnonzero(sg.train_mask))
            cpu = cpu_baseline(args, sg, args.cpu_sample_s, norms)
        F = sg.features.shape[1]
        fb = 4 * ((F + 31) // 32) if tr.dg.xbits else 4 * F  # feature bytes per row
        gat_us = gather[0]["avg_us"] if gather else None
        out = {
            "metric": METRIC,
            "value": round(1000.0 / ms_per_step, 3),
            "unit": "iters/s",
            "n_gpus": world,
            "steps": K,
            "warmup": W,
            "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32" if args.dtype == "float32" else "f64",
            "data": f"synthetic ({args.shape}-shaped O(m) SBM, random-init weights)",
            "config": bench_config(args, sg.n_nodes, sg.nnz, F),
            "pipeline": {"plans_per_sampler_launch": T * n_my, "lookahead_iters": T,
                         "sampler_streams": S, "workers_this_rank": n_my,
                         "timing": "steady state: the warm-up samples the region's first "
                                   f"{S} plan groups, the region samples the {S} groups after "
                                   "it (equal work), events on the main stream after joining "
                                   "the sampler streams; max over ranks"},
            "remote_nodes_per_iter": round(remote_per_iter, 2),
            "input_layer_remote_rows_per_iter": s0_remote,
            "sampled_nodes_per_s": round(sampled_nodes / (ms_per_step * 1e-3), 1),
            "exchange": {
                "remote_input_rows_per_iter": s0_remote,
                "bytes_per_iter": int(round(s0_remote * (fb + 4))),
                "feature_rows": ("bit-packed multi-hot, %d B per row" % fb if tr.dg.xbits
                                 else "fp32, %d B per row" % fb),
                "input_rows_per_iter": s0_rows,
                "path": ("NVLink P2P: the layer-0 SpMM (k_spmm_in_b, gather fused) reads remote "
                         "rows from CUDA-IPC-mapped peer shards" if world > 1 else
                         "one rank holds every feature row: remote rows are read from local "
                         "HBM (no link traffic)"),
                "gather_us_per_launch": gat_us,
                "gather_gbs": (round(s0_rows * fb / (gat_us * 1e-6) / 1e9, 2)
                               if gat_us else None),
                "remote_link_gbs": (round(s0_remote * (fb + 4) / (gat_us * 1e-6) / 1e9, 2)
                                    if gat_us and world > 1 else None)},
            "allreduce": ar,
            "gpu_launches": int(launches),
            "host_enqueue_ms_per_step": round(host_ms / K, 4),
            "stages_ms_per_iter": {"sample": round(samp / n_it, 4),
                                   "gcn_fwd_bwd_step": round(float(np.median(comp_ms)), 4)},
            "roofline": {"bound": top["bound"], "kernel": top["kernel"],
                         "achieved": top["achieved"], "peak": top["peak"], "unit": top["unit"],
                         "frac": top["frac"], **ncu_traffic(top["kernel"], args.shape),
                         **{k_: top[k_] for k_ in ("frac_of_3xtf32_peak", "peak_note") if k_ in top},
                         "per_launch": top["per_launch"], "avg_launch_us": top["avg_us"],
                         "share_of_step": top["share"],
                         "dominant_kernel": dominant,
                         "timing": "CUDA events around every launch of every kernel on its "
                                   "stream, over the K timed steps replayed with the stages "
                                   "serialised (as the ncu launch list sees them); share = "
                                   "kernel total / all kernels' total",
                         "peak_source": "MEASURED_PEAKS.json (burst: kernels timed alone)"},
            "kernels": kern,
            "sampler_stage": {"achieved_gbs": round(achieved, 2), "frac": round(achieved / hbm, 5),
                              "algorithmic_bytes": int(alg_bytes), "duration_ms": round(samp, 4),
                              "plans": n_it * n_my,
                              "bytes_model": "SURVEY §8(d) verbatim, summed over the plans' "
                                             "layers (statistics of the sampled plans)"},
            "e2e": {"value": round(1000.0 * K / e2e_ms, 3), "unit": "iters/s",
                    "h2d_bytes_per_step": int(h2d[0] // K), "d2h_bytes_per_step": 8 * n_my,
                    "timing": "host clock around Trainer.run over the K steps (steady state, "
                              "like the device region), every loss read on the host"},
            "clocks": clk.summary(),
            "graph_build_s": round(t_gen, 2),
        }
        if cpu is not None:
            out["cpu_baseline"] = cpu
        print(json.dumps(out), flush=True)
    tr.close()
    if dist is not None:
        dist.destroy_process_group()
    return out


def prepare_graphs(tr, lib, sample_fn, T, n_my, sizes):
    """Capture (without replaying) the sampler launch sequence for every group size and
    the batched training step at every group offset, in every plan arena."""
    import torch
    from paper_2101_07706_b200._native import check
    from ctypes import c_uint64, POINTER
    sizes = sorted({s for s in sizes if s > 0})
    check(lib.skg_set_capture_only(1))
    try:
        for b, (ps, gcn) in enumerate(tr.bufs):
            for n in sizes:
                sample_fn(0, n, b)
            for gi in range(T):
                check(lib.skg_gcn_step_batch(gcn, gi * n_my, n_my,
                                             tr.wp.ctypes.data_as(POINTER(c_uint64)),
                                             tr.gp.ctypes.data_as(POINTER(c_uint64)), 0,
                                             tr.losses[0].data_ptr(), tr.stream))
    finally:
        check(lib.skg_set_capture_only(0))
    torch.cuda.synchronize()


def kernel_table(lib, steps_fn, W, K, stats, tr, T, peaks, saint, budget):
    """Event-time every kernel over the K timed steps (replayed by steps_fn, one pass with
    every launch bracketed) and relate each to its algorithmic bytes (HBM-bound sampler
    kernels, SURVEY §8(d) terms) or flops (tensor-core GEMMs), per launch name (the GEMM's
    template instantiations separately)."""
    import torch
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    tflops = float(peaks.get("bf16_tflops", 1590.0))
    L = N_LAYERS
    n_it = max(1, len(stats) // max(tr.n_my, 1))
    launches_per_group = 1 if saint else L
    # §8(d) bytes of the sampled group (n_it iterations' plans), per sampler launch
    models = ({} if saint else
              {k_: v / launches_per_group for k_, v in kernel_bytes_8d(stats, budget).items()})
    dims = tr.dims
    rows = [sum(int(st[0 if saint else L - 1 - l, 0]) for st in stats) / n_it for l in range(L)]
    # per training step (all of the rank's slots): SpMM per call, SURVEY §8(d)
    # 8*nnz + 4*(rows+1) + 4*cols*d + 4*rows*d; the layer-0 gather 4*F*|S_0| + 4*|S_0|
    def lay(l, c):
        return sum(int(st[0 if saint else L - 1 - l, c]) for st in stats) / n_it

    def spmm_bytes(l):
        r, c, z = lay(l, 0), lay(l, 2), lay(l, 3)
        return 8 * z + 4 * (r + tr.n_my) + 4 * c * dims[l] + 4 * r * dims[l]

    inner = list(range(1, L))
    # layer 0: the gather fused into the SpMM; its source rows are feature rows
    fb = 4 * ((dims[0] + 31) // 32) if tr.dg.xbits else 4 * dims[0]
    r0, c0, z0 = lay(0, 0), lay(0, 2), lay(0, 3)
    models["k_spmm_in_b<bits>" if tr.dg.xbits else "k_spmm_in_b"] = (
        8 * z0 + 4 * (r0 + tr.n_my) + fb * c0 + 4 * c0 + 4 * r0 * dims[0])
    models["k_spmm_b<F,0>"] = spmm_bytes(0)
    if inner:
        models["k_spmm_b<F,1>"] = sum(spmm_bytes(l) for l in inner) / len(inner)
        models["k_spmm_b<T,1,0>"] = sum(spmm_bytes(l) for l in inner) / len(inner)
    torch.cuda.synchronize()
    lib.skg_profile_start(b"*")
    steps_fn(W, K)
    buf = C.create_string_buffer(1 << 16)
    lib.skg_profile_table(buf, len(buf))
    table = []
    for line in buf.value.decode().splitlines():
        name, cnt, tot = line.rsplit(" ", 2)
        table.append((name, int(cnt), float(tot)))
    all_ms = sum(t for _, _, t in table)
    out = []
    for name, cnt, tot in table:
        avg_s = tot / cnt * 1e-3
        row = {"kernel": name, "launches": cnt, "total_ms": round(tot, 4),
               "avg_us": round(avg_s * 1e6, 2), "share": round(tot / all_ms, 4)}
        base = name.split("<")[0]
        if name in models:
            base = name  # per-instantiation model (SpMM variants)
        if base in ("k_gemm_tc", "k_gemm_tc_p") and "@l" in name:
            # every GEMM of GCN layer l (forward U W, dW = U^T G, dX = G W^T) contracts
            # rows_l x d_l x d_{l+1}: 2 * rows_l * d_l * d_{l+1} algorithmic flops per launch
            l = int(name.rsplit("@l", 1)[1])
            per = 2.0 * rows[l] * dims[l] * dims[l + 1]
            ach = per / avg_s / 1e12
            row.update({"bound": "tensor", "unit": "TFLOP/s", "peak": tflops,
                        "per_launch": {"flops": int(per)}, "achieved": round(ach, 2),
                        "frac": round(ach / tflops, 5),
                        # each algorithmic flop is 3 TF32 MMA flops at half the bf16 rate
                        "frac_of_3xtf32_peak": round(ach / (tflops / 6.0), 5),
                        "peak_note": "3xTF32 ceiling = measured bf16 / 2 (TF32 rate) / 3 (passes)"})
        elif base in models:
            # the statistics cover n_it iterations per launch; the replayed K steps run
            # K / ceil(K / T) iterations per launch on average (a partial last group)
            per = models[base]
            if not base.startswith(("k_gather", "k_spmm")):  # sampler launches: per group
                per = per * (K / -(-K // T)) / n_it
            ach = per / avg_s / 1e9
            row.update({"bound": "hbm", "unit": "GB/s", "peak": hbm, "per_launch": {"bytes": int(per)},
                        "achieved": round(ach, 2), "frac": round(ach / hbm, 5)})
        else:
            row.update({"bound": "latency", "unit": None, "peak": None, "per_launch": None,
                        "achieved": None, "frac": None})
        out.append(row)
    out.sort(key=lambda r: -r["total_ms"])
    return out, all_ms


def ncu_traffic(kernel_label, shape="reddit"):
    """DRAM bytes per launch of the roofline kernel from the committed ncu --set full
    extract (profiles/ncu_traffic.json, tools/ncu_traffic.py; cold-cache replay, so an upper
    bound on the in-step traffic); null when the kernel was not captured on this shape
    (entries without a "shape" were captured on the default Reddit workload)."""
    path = ROOT / "profiles" / "ncu_traffic.json"
    base = kernel_label.split(" ")[0].split("<")[0]
    try:
        table = json.loads(path.read_text())
    except (OSError, ValueError):
        return {"traffic": None}
    hits = [k for k in table if (k == base or k.startswith(base + "_"))
            and table[k].get("shape", "reddit") == shape]
    if not hits:
        return {"traffic": None}
    t = table[hits[0]]
    return {"traffic": int(t["dram_bytes"]), "traffic_source": f"profiles/ncu_traffic.json ({hits[0]}, "
            f"mean of {t['launches']} ncu --set full launches, cold cache)"}


# ---------------------------------------------------------------------------- CPU oracle
def _oracle_setup(args, sg, saint_norms=None):
    """The oracle (a CPU restatement of the reference) on the same synthetic graph.
    GraphSAINT plans take precomputed training-set column norms (the reference computes
    them once per run, training.py:462-464): `saint_norms` or the oracle's own."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import skewgcn_oracle as O
    og = O.Graph(n_nodes=sg.n_nodes, offsets=sg.offsets, neighbors=sg.neighbors.astype(np.int64),
                 weights=sg.weights, normalized=True, features=sg.features.astype(np.float64),
                 labels=sg.labels, train_mask=sg.train_mask, val_mask=sg.val_mask)
    part = O.partition_nodes(sg.n_nodes, args.workers, "random", seed=1)
    dims = [sg.features.shape[1]] + [args.hidden] * (N_LAYERS - 1) + [sg.n_classes]
    ws = O.init_model(dims, 0)
    saint = args.sampler == "saint"
    cfg = O.SamplerConfig(budget=args.subgraph if saint else args.budget, skew_constant=args.D,
                          mode=args.mode)
    wt = [np.flatnonzero(og.train_mask & (part.owner == w)) for w in range(args.workers)]
    ctx = {"O": O, "og": og, "part": part, "ws": ws, "cfg": cfg, "wt": wt, "args": args}
    if saint:
        train = np.flatnonzero(og.train_mask)
        ctx["train"] = train
        if args.mode != "local":
            ctx["norms"] = saint_norms if saint_norms is not None else O.column_norms(og, train, train)
    return ctx


def _oracle_worker_iter(ctx, it, w):
    O, og, args = ctx["O"], ctx["og"], ctx["args"]
    prng = O.spawn_rng(0, "plan", 0, it, w)
    if args.sampler == "saint":
        plan = O.saint_plan(og, ctx["part"], w, ctx["train"], args.subgraph, ctx["cfg"], N_LAYERS,
                            prng, norms=ctx.get("norms"))
    else:
        brng = O.spawn_rng(0, "batch", 0, it, w)
        wt = ctx["wt"][w]
        batch = O.node_set(brng.choice(wt, size=min(args.batch, len(wt)), replace=False))
        plan = O.ladies_plan(og, ctx["part"], w, batch, ctx["cfg"], N_LAYERS, prng)
    loss, grads = O.loss_and_backward(ctx["ws"], plan, og.features, og.labels)
    return loss


def cpu_baseline(args, sg, budget_s, saint_norms=None):
    """The oracle port timed on this host: whole worker-iterations until ~budget_s."""
    from threadpoolctl import threadpool_limits
    ctx = _oracle_setup(args, sg, saint_norms)
    times = []
    t_all = time.perf_counter()
    w = 0
    with threadpool_limits(limits=1):  # one core: BLAS single-threaded too
        while True:
            t0 = time.perf_counter()
            _oracle_worker_iter(ctx, 0, w % args.workers)
            times.append(time.perf_counter() - t0)
            w += 1
            if time.perf_counter() - t_all > budget_s and w >= 2:
                break
    per_worker = float(np.median(times))
    it_s = 1.0 / (args.workers * per_worker)
    return {"value": round(it_s, 5), "unit": "iters/s", "cores": 1, "kind": "port",
            "sample": f"{len(times)} worker-iterations (plan + fwd/bwd) of the k={args.workers} "
                      f"iteration, median {per_worker:.3f} s; iters/s = 1/(k * median)",
            "threads_note": f"one thread (BLAS limited by threadpoolctl); os.cpu_count()={os.cpu_count()}"}


_REF_CTX = None


def _ref_task(a):
    return _oracle_worker_iter(_REF_CTX, a[0], a[1])


_REF_LIMITS = None


def _ref_worker_init(threads):
    # BLAS threads per worker process: cores / processes (an unlimited pool per process
    # oversubscribes the host ~k-fold and runs the reference ~8x slower)
    global _REF_LIMITS
    from threadpoolctl import threadpool_limits
    _REF_LIMITS = threadpool_limits(limits=threads)


def run_reference(args):
    """The reference arm; GraphSAINT / LADIES softmax configurations only (the reference
    has no multi-label loss).

    The reference algorithm (oracle port) on the host: each step is one full iteration,
    its k worker-iterations (plan + forward/backward) run in parallel worker processes
    (fork, copy-on-write graph) on all usable host cores."""
    global _REF_CTX
    import multiprocessing as mp
    world, rank, local = dist_setup(args)
    if rank != 0:
        return None
    if args.shape.startswith("youtube"):
        out = {"impl": "reference", "unavailable": "the reference has no multi-label (BCE) loss"}
        print(json.dumps(out), flush=True)
        return out
    sg = shape_info(args.shape).make_shaped_graph(args.shape, seed=0, device=None)
    _REF_CTX = _oracle_setup(args, sg)
    usable = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    procs = max(1, min(args.workers, usable))
    per_proc = max(1, usable // procs)
    cores = procs * per_proc
    pool = (mp.get_context("fork").Pool(procs, initializer=_ref_worker_init, initargs=(per_proc,))
            if procs > 1 else None)
    if pool is None:
        _ref_worker_init(per_proc)

    def step(it):
        tasks = [(it, w) for w in range(args.workers)]
        if pool is None:
            return [_ref_task(t) for t in tasks]
        return pool.map(_ref_task, tasks, chunksize=1)

    for s in range(args.warmup):
        step(s)
    times = []
    for s in range(args.steps):
        t0 = time.perf_counter()
        step(args.warmup + s)
        times.append(time.perf_counter() - t0)
    if pool is not None:
        pool.close()
        pool.join()
    per_step = float(np.mean(times))
    it_s = 1.0 / per_step
    out = {"metric": METRIC, "value": round(it_s, 5), "unit": "iters/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(per_step * 1e3, 2), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": f"synthetic ({args.shape}-shaped O(m) SBM, random-init weights)",
           "config": bench_config(args, sg.n_nodes, sg.nnz, sg.features.shape[1]),
           "impl": "reference",
           "cpu_baseline": {"value": round(it_s, 5), "unit": "iters/s", "cores": cores, "kind": "port",
                            "sample": f"{args.steps} iterations, each the k={args.workers} "
                                      f"worker-iterations in {procs} parallel processes x "
                                      f"{per_proc} BLAS threads; iters/s = 1/mean step time"},
           "e2e": {"value": round(it_s, 5), "unit": "iters/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    a = parse()
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        sys.exit(spawn_ranks(a))  # one rank per GPU (torch.distributed.run on 127.0.0.1)
    if int(os.environ.get("WORLD_SIZE", "1")) != a.gpus:
        sys.stderr.write(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}\n")
        sys.exit(2)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
