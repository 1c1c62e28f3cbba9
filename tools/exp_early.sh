# GEMM stage 0 issued before the setup sync: GEMM / shaped / graph tests, then the step A/B
mkdir -p gpurun_out/exp10
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_shaped.py tests/test_gpu_epilogue.py tests/test_gpu_graphs.py -x -q > gpurun_out/exp10/tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/exp10/tests.txt
tail -2 gpurun_out/exp10/tests.txt
for rep in 1 2 3; do
  for e in 1 0; do
    SKG_GEMM_EARLY=$e timeout 300 python bench.py --no-cpu-baseline > gpurun_out/exp10/e${e}_r$rep.json 2> gpurun_out/exp10/e${e}_r$rep.err
  done
done
for e in 1 0; do
  SKG_GEMM_EARLY=$e timeout 300 python bench.py --shape youtube --no-cpu-baseline > gpurun_out/exp10/yt_e$e.json 2> gpurun_out/exp10/yt_e$e.err
done
