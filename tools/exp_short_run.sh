# the driver's short run (--steps 20 --warmup 5) at several look-ahead depths
mkdir -p gpurun_out/exp5
for rep in 1 2; do
  for a in 2 3 4 5; do
    timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --ahead $a --no-cpu-baseline > gpurun_out/exp5/a${a}_r$rep.json 2> gpurun_out/exp5/a${a}_r$rep.err
  done
done
