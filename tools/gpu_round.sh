# round-end style evidence run: GPU suite, smoke, bench (N=1), reference arm, launch list,
# ncu --set full of the top sampler / GCN kernels; outputs under gpurun_out/$SKG_TAG
set -x
O=gpurun_out/${SKG_TAG:-round}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref.json 2> $O/ref.err
timeout 600 python bench.py --shape youtube --no-cpu-baseline > $O/bench_youtube.json 2> $O/bench_youtube.err
timeout 600 python bench.py --shape amazon --sampler saint --no-cpu-baseline > $O/bench_amazon.json 2> $O/bench_amazon.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $O/launches.csv python bench.py --steps 10 --warmup 5 --no-cpu-baseline > $O/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_lad_range|k_cs_maps|k_draw_dedup|k_cs_walk|k_pw_leaves|k_lad_finish|k_heavy_fold|k_gemm_tc|k_spmm_in_b|k_spmm_b" \
  --launch-skip 40 --launch-count 24 -o $O/full -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/full.ncu-rep > $O/full_summary.txt 2>&1
tail -3 $O/pytest_gpu.log
