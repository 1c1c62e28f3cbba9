# one build -> measure iteration on the B200: sampler/GCN parity tests, the bench line,
# optionally an ncu --set full capture of kernels matching $SKG_NCU (one layer's launches)
O=gpurun_out/${SKG_TAG:-iter}
mkdir -p $O
timeout 900 python -m pytest ${SKG_TESTS:-tests/test_gpu_parity.py tests/test_gpu_shaped.py} -x -q > $O/tests.log 2>&1
echo "tests rc $?" >> $O/tests.log
tail -2 $O/tests.log
timeout 600 python bench.py --no-cpu-baseline ${SKG_BENCH_ARGS} > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "stages", d.get("stages_ms_per_iter"), "sampler frac", d.get("sampler_stage", {}).get("frac"))
for k in d.get("kernels", [])[:16]:
    print(f'{k["kernel"]:28s} {k["avg_us"]:8.2f} us  share {k["share"]:.3f}')
PY
if [ -n "$SKG_NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$SKG_NCU" \
    --launch-skip ${SKG_NCU_SKIP:-18} --launch-count ${SKG_NCU_COUNT:-9} -o $O/full -f \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
  python tools/ncu_summary.py $O/full.ncu-rep > $O/summary.txt 2>&1
  cat $O/summary.txt
fi
