# ncu --set full capture of one 24-plan layer of each top sampler kernel (bench workload),
# then the new shaped / F1 GPU tests
set -x
O=gpurun_out/${SKG_TAG:-r2b}
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_lad_range|k_cs_maps|k_draw_dedup|k_cs_walk|k_pw_leaves|k_lad_finish|k_heavy_fold|k_heavy_scan|k_pw_top" \
  --launch-skip 18 --launch-count 9 -o $O/sampler_full -f \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
ncu -i $O/sampler_full.ncu-rep --page raw --csv > $O/sampler_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/sampler_full.ncu-rep > $O/sampler_summary.txt 2>&1
if [ -n "$SKG_TESTS" ]; then
  SKG_F1_OUT=$O/f1.jsonl timeout 1200 python -m pytest $SKG_TESTS -x -q -s > $O/tests.log 2>&1
  echo "tests rc $?" >> $O/tests.log
fi
