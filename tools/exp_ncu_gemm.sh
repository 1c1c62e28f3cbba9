# ncu --set full of the LADIES step's tensor-core GEMMs (TMA-store epilogue)
mkdir -p gpurun_out/exp9
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_gemm_tc$' --launch-skip 60 -c 6 -o gpurun_out/exp9/gemm -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/exp9/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/exp9/gemm.ncu-rep > gpurun_out/exp9/summary.txt 2>&1
cat gpurun_out/exp9/summary.txt
