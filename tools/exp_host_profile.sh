# host-side profile of the timed loop, a sampler-only run, and an ncu capture of the
# GraphSAINT GEMMs (non-persistent k_gemm_tc: the dW launches)
set -x
mkdir -p gpurun_out/exp2
SKG_BENCH_PROFILE=1 timeout 600 python bench.py --steps 400 --no-cpu-baseline > gpurun_out/exp2/bench_prof.json 2> gpurun_out/exp2/bench_prof.err
SKG_BENCH_SAMPLER_ONLY=1 timeout 600 python bench.py --steps 400 --no-cpu-baseline > gpurun_out/exp2/bench_sampler_only.json 2> gpurun_out/exp2/bench_sampler_only.err
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_gemm_tc$' --launch-skip 40 -c 3 -o gpurun_out/exp2/amazon_gemm python bench.py --shape amazon --sampler saint --steps 10 --no-cpu-baseline > gpurun_out/exp2/ncu.log 2>&1
