"""BASELINE configs[4]: Full vs Local vs skewed (D in {4, 8, 16, 32}) on the Reddit-shaped graph
with k = 8 workers: iters/s and communicated nodes per iteration (the reference's ledger) on
one GPU.  Writes one JSON line per setting to stdout."""
import json
import subprocess
import sys

steps = sys.argv[1] if len(sys.argv) > 1 else "200"
runs = [("full", 0.0), ("local", 0.0)] + [("skewed", d) for d in (4.0, 8.0, 16.0, 32.0)]
for mode, D in runs:
    out = subprocess.run([sys.executable, "bench.py", "--no-cpu-baseline", "--steps", steps, "--mode", mode,
                          "--D", str(D)], capture_output=True, text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")]
    if not line:
        print(json.dumps({"mode": mode, "D": D, "error": out.stderr[-400:]}), flush=True)
        continue
    d = json.loads(line[-1])
    print(json.dumps({"mode": mode, "D": D, "iters_per_s": d["value"], "e2e_iters_per_s": d["e2e"]["value"],
                      "remote_nodes_per_iter": d["remote_nodes_per_iter"],
                      "input_layer_remote_rows_per_iter": d["input_layer_remote_rows_per_iter"],
                      "sampled_nodes_per_s": d["sampled_nodes_per_s"],
                      "stages_ms_per_iter": d["stages_ms_per_iter"]}), flush=True)
