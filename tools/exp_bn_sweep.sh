# GEMM N tile with the TMA-store epilogue
mkdir -p gpurun_out/exp7
for rep in 1 2; do
  for bn in 0 64 256; do
    if [ $bn = 0 ]; then unset SKG_GEMM_BN; else export SKG_GEMM_BN=$bn; fi
    timeout 300 python bench.py --no-cpu-baseline > gpurun_out/exp7/bn${bn}_r$rep.json 2> gpurun_out/exp7/bn${bn}_r$rep.err
  done
done
unset SKG_GEMM_BN
for bn in 0 64 256; do
  if [ $bn = 0 ]; then unset SKG_GEMM_BN; else export SKG_GEMM_BN=$bn; fi
  timeout 300 python bench.py --shape youtube --no-cpu-baseline > gpurun_out/exp7/yt_bn${bn}.json 2> gpurun_out/exp7/yt_bn${bn}.err
done
