# vectorised slot reduction: GPU suite (incl. the epilogue test) and the step
mkdir -p gpurun_out/exp8
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp8/suite.txt 2>&1; echo "pytest rc $?" >> gpurun_out/exp8/suite.txt
tail -3 gpurun_out/exp8/suite.txt
for rep in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/exp8/reddit_r$rep.json 2> gpurun_out/exp8/reddit_r$rep.err
done
timeout 300 python bench.py --shape youtube --no-cpu-baseline > gpurun_out/exp8/youtube.json 2> gpurun_out/exp8/youtube.err
