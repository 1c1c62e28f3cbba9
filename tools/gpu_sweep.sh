# bench variants on one box: each line of $SKG_SWEEP is a set of bench.py arguments
O=gpurun_out/${SKG_TAG:-sweep}
mkdir -p $O
i=0
echo "$SKG_SWEEP" | tr ';' '\n' | while read -r args; do
  [ -z "$args" ] && continue
  i=$((i+1))
  timeout 600 python bench.py --no-cpu-baseline $args > $O/b$i.json 2> $O/b$i.err
  python - "$O/b$i.json" "$args" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f'{sys.argv[2]:40s} value {d["value"]:9.2f} e2e {d["e2e"]["value"]:9.2f} stages {d.get("stages_ms_per_iter")}')
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
