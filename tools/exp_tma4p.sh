# 4D MN-major boxes also in the persistent GEMM (GraphSAINT): kernel tests, Amazon A/B
mkdir -p gpurun_out/exp15
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_epilogue.py tests/test_gpu_graphs.py tests/test_gpu_experiment.py -x -q > gpurun_out/exp15/tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/exp15/tests.txt
tail -2 gpurun_out/exp15/tests.txt
for rep in 1 2; do
  for t in 1 2; do
    SKG_GEMM_TMA4=$t timeout 300 python bench.py --shape amazon --sampler saint --no-cpu-baseline > gpurun_out/exp15/am_t${t}_r$rep.json 2> gpurun_out/exp15/am_t${t}_r$rep.err
  done
done
