# number of K chunks loaded before the GEMM's setup sync
mkdir -p gpurun_out/exp16
SKG_GEMM_EARLY=2 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_epilogue.py -x -q > gpurun_out/exp16/tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/exp16/tests.txt
tail -2 gpurun_out/exp16/tests.txt
for rep in 1 2; do
  for e in 1 2 3; do
    SKG_GEMM_EARLY=$e timeout 300 python bench.py --no-cpu-baseline > gpurun_out/exp16/e${e}_r$rep.json 2> gpurun_out/exp16/e${e}_r$rep.err
  done
done
for e in 1 2 3; do
  SKG_GEMM_EARLY=$e timeout 300 python bench.py --shape youtube --no-cpu-baseline > gpurun_out/exp16/yt_e$e.json 2> gpurun_out/exp16/yt_e$e.err
done
