# PDL on every kernel, sampler kernels triggering their dependents at their end
mkdir -p gpurun_out/exp13
SKG_PDL=1 timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/exp13/suite_pdl1.txt 2>&1; echo "pytest rc $?" >> gpurun_out/exp13/suite_pdl1.txt
tail -2 gpurun_out/exp13/suite_pdl1.txt
for rep in 1 2 3; do
  for p in 1 2; do
    SKG_PDL=$p timeout 300 python bench.py --no-cpu-baseline > gpurun_out/exp13/p${p}_r$rep.json 2> gpurun_out/exp13/p${p}_r$rep.err
  done
done
for p in 1 2; do
  SKG_PDL=$p timeout 300 python bench.py --shape youtube --no-cpu-baseline > gpurun_out/exp13/yt_p$p.json 2> gpurun_out/exp13/yt_p$p.err
  SKG_PDL=$p timeout 300 python bench.py --shape amazon --sampler saint --no-cpu-baseline > gpurun_out/exp13/am_p$p.json 2> gpurun_out/exp13/am_p$p.err
done
