# bench under several environments on one box: $SKG_SWEEP = "ENV=.. ENV2=..;ENV=..;..." ("-" = none)
O=gpurun_out/${SKG_TAG:-esweep}
mkdir -p $O
i=0
echo "$SKG_SWEEP" | tr ';' '\n' | while read -r envs; do
  [ -z "$envs" ] && continue
  i=$((i+1))
  if [ "$envs" = "-" ]; then e=""; else e="$envs"; fi
  env $e timeout 600 python bench.py --no-cpu-baseline $SKG_BENCH_ARGS > $O/b$i.json 2> $O/b$i.err
  python - "$O/b$i.json" "$envs" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ks = {k["kernel"]: k["avg_us"] for k in d.get("kernels", [])}
    top = sorted(d.get("kernels", []), key=lambda k: -k["share"])[:6]
    print(f'{sys.argv[2]:40s} value {d["value"]:9.2f} e2e {d["e2e"]["value"]:9.2f} stages {d.get("stages_ms_per_iter")}')
    print("   ", ", ".join(f'{k["kernel"]} {k["avg_us"]}' for k in top))
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
