"""bench.py's contract: the reference arm runs the CPU oracle without mapping libskg.so and
prints the same `config` dict as the CUDA arm; `--gpus N` launches N ranks itself (checked
on the GPU box with ranks sharing its one GPU over gloo)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

_REF = r"""
import runpy, sys, json, io, contextlib
sys.argv = ["bench.py", "--impl", "reference", "--shape", "cora", "--steps", "2", "--warmup", "1"]
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    runpy.run_path("bench.py", run_name="__main__")
line = [l for l in buf.getvalue().splitlines() if l.startswith("{")][-1]
maps = open("/proc/self/maps").read()
print(json.dumps({"line": json.loads(line), "libskg": "libskg" in maps,
                  "pkg": any(m.startswith("paper_2101_07706_b200") for m in sys.modules)}))
"""


def test_reference_arm_no_native_library_same_config():
    r = subprocess.run([sys.executable, "-c", _REF], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert not out["libskg"], "the reference arm mapped libskg.so"
    assert not out["pkg"], "the reference arm imported the CUDA package"
    line = out["line"]
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    sys.path.insert(0, str(ROOT))
    import bench
    args = bench.parse_args(["--shape", "cora"])
    sg = bench.shape_info("cora").make_shaped_graph("cora", seed=0, with_features=False)
    assert line["config"] == bench.bench_config(args, sg.n_nodes, sg.nnz, 1433)
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_bench_spawns_ranks_gloo():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks (gloo: they share the box's
    GPU) and prints one line with n_gpus 2, the exchange and all-reduce fields."""
    env = dict(os.environ, SKG_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "6", "--warmup", "3",
                        "--shape", "reddit_s", "--no-cpu-baseline"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["steps"] == 6 and out["warmup"] == 3
    assert out["pipeline"]["workers_this_rank"] == 4
    assert out["pipeline"]["plans_per_sampler_launch"] == 40  # ceil(40 / 4) iterations ahead
    assert out["exchange"]["remote_input_rows_per_iter"] > 0
    assert out["allreduce"]["bytes"] > 0 and out["allreduce"]["backend"] == "gloo"
    assert out["e2e"]["value"] > 0 and out["gpu_launches"] > 0
