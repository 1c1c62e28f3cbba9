set -x
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2a/ref.json 2> gpurun_out/r2a/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r2a/launches.csv python bench.py --steps 8 --warmup 4 --no-cpu-baseline > gpurun_out/r2a/ncu_bench.log 2>&1
tail -3 gpurun_out/r2a/pytest_gpu.log
