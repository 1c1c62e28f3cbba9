# TMA-store GEMM epilogue: GPU suite, then the step with and without it
mkdir -p gpurun_out/exp6
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp6/suite.txt 2>&1; echo "pytest rc $?" >> gpurun_out/exp6/suite.txt
tail -3 gpurun_out/exp6/suite.txt
for rep in 1 2; do
  for t in 1 0; do
    SKG_GEMM_TMA_STORE=$t timeout 300 python bench.py --no-cpu-baseline > gpurun_out/exp6/reddit_t${t}_r$rep.json 2> gpurun_out/exp6/reddit_t${t}_r$rep.err
  done
done
for t in 1 0; do
  SKG_GEMM_TMA_STORE=$t timeout 300 python bench.py --shape youtube --no-cpu-baseline > gpurun_out/exp6/youtube_t$t.json 2> gpurun_out/exp6/youtube_t$t.err
  SKG_GEMM_TMA_STORE=$t timeout 300 python bench.py --shape amazon --sampler saint --no-cpu-baseline > gpurun_out/exp6/amazon_t$t.json 2> gpurun_out/exp6/amazon_t$t.err
done
