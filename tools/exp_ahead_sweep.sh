# look-ahead depth (plans per sampler launch = ahead x workers) and sampler stream count
mkdir -p gpurun_out/exp4
for a in 4 5 6 7 8 10; do
  for s in 2 3; do
    timeout 300 python bench.py --steps 400 --ahead $a --streams $s --no-cpu-baseline > gpurun_out/exp4/a${a}_s${s}.json 2> gpurun_out/exp4/a${a}_s${s}.err
  done
done
timeout 600 python bench.py --shape youtube --no-cpu-baseline > gpurun_out/exp4/youtube.json 2> gpurun_out/exp4/youtube.err
timeout 600 python bench.py --shape amazon --sampler saint --no-cpu-baseline > gpurun_out/exp4/amazon.json 2> gpurun_out/exp4/amazon.err
