# range-expand CTA timelines seen from several warps (phase-1 balance across warps)
mkdir -p gpurun_out/exp3
for t in 0 96 320 544 800 1023; do
  SKG_FR_TRACE=gpurun_out/exp3/tr_$t.json SKG_FR_TRACE_THREAD=$t timeout 300 python bench.py --steps 50 --no-cpu-baseline > gpurun_out/exp3/b_$t.json 2> gpurun_out/exp3/b_$t.err
done
