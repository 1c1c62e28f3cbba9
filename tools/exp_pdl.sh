# PDL on the GCN chain with the GEMM's late trigger: correctness under PDL, then the step A/B
mkdir -p gpurun_out/exp12
SKG_PDL=2 timeout 900 python -m pytest tests/test_gpu_shaped.py tests/test_gpu_graphs.py tests/test_gpu_epilogue.py -x -q > gpurun_out/exp12/tests_pdl2.txt 2>&1; echo "pytest rc $?" >> gpurun_out/exp12/tests_pdl2.txt
tail -2 gpurun_out/exp12/tests_pdl2.txt
for rep in 1 2 3; do
  for p in 2 0; do
    SKG_PDL=$p timeout 300 python bench.py --no-cpu-baseline > gpurun_out/exp12/p${p}_r$rep.json 2> gpurun_out/exp12/p${p}_r$rep.err
  done
done
for p in 2 0; do
  SKG_PDL=$p timeout 300 python bench.py --shape youtube --no-cpu-baseline > gpurun_out/exp12/yt_p$p.json 2> gpurun_out/exp12/yt_p$p.err
done
for p in 2 0; do
  SKG_PDL=$p timeout 300 python bench.py --shape amazon --sampler saint --no-cpu-baseline > gpurun_out/exp12/am_p$p.json 2> gpurun_out/exp12/am_p$p.err
done
