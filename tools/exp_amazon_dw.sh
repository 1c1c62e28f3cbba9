set -x
mkdir -p gpurun_out/exp1
SKG_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/exp1/bench_2rank_gloo.json 2> gpurun_out/exp1/bench_2rank_gloo.err
for ks in 0 3 4 6 8; do
  if [ $ks = 0 ]; then unset SKG_GEMM_KSPLIT; else export SKG_GEMM_KSPLIT=$ks; fi
  timeout 600 python bench.py --shape amazon --sampler saint --steps 100 --no-cpu-baseline > gpurun_out/exp1/amazon_ks$ks.json 2> gpurun_out/exp1/amazon_ks$ks.err
done
unset SKG_GEMM_KSPLIT
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_gemm_tc<true' --launch-skip 20 -c 2 -o gpurun_out/exp1/amazon_dw python bench.py --shape amazon --sampler saint --steps 10 --no-cpu-baseline > gpurun_out/exp1/ncu.log 2>&1
