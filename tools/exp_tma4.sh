# MN-major GEMM operands in one 4D TMA box per stage: GEMM / shaped / graph tests, step A/B
mkdir -p gpurun_out/exp14
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_shaped.py tests/test_gpu_epilogue.py tests/test_gpu_graphs.py tests/test_gpu_parity.py -x -q > gpurun_out/exp14/tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/exp14/tests.txt
tail -2 gpurun_out/exp14/tests.txt
for rep in 1 2 3; do
  for t in 1 0; do
    SKG_GEMM_TMA4=$t timeout 300 python bench.py --no-cpu-baseline > gpurun_out/exp14/t${t}_r$rep.json 2> gpurun_out/exp14/t${t}_r$rep.err
  done
done
for t in 1 0; do
  SKG_GEMM_TMA4=$t timeout 300 python bench.py --shape youtube --no-cpu-baseline > gpurun_out/exp14/yt_t$t.json 2> gpurun_out/exp14/yt_t$t.err
  SKG_GEMM_TMA4=$t timeout 300 python bench.py --shape amazon --sampler saint --no-cpu-baseline > gpurun_out/exp14/am_t$t.json 2> gpurun_out/exp14/am_t$t.err
done
