# round-end evidence: bench lines of every config, the cfg2 launch list, and
# ncu --set full of the dominant kernels (cfg2 step kernels, cfg4 l chains,
# T1279 analysis) -> gpurun_out/
mkdir -p gpurun_out
STEPS=20 bash scripts/gpu_bench_configs.sh
SWX_FORCE_COMM=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --config cfg4 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_cfg4_comm.json 2> gpurun_out/bench_cfg4_comm.err; echo "cfg4 comm rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --profile"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
for K in synth_kernel grid_sq1 analysis_tab rexi_lg_mm; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1; echo "$K rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:rexi_l_kernel -s 1 -c 1 -o gpurun_out/prof_rexi_l_cfg4 python bench.py --config cfg4 --steps 1 --warmup 1 --profile --no-cpu --no-e2e > gpurun_out/ncu_l4.log 2>&1; echo "l cfg4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:analysis_col -c 1 -o gpurun_out/prof_analysis_col python scripts/rt1279.py > gpurun_out/ncu_acol.log 2>&1; echo "acol rc=$?"
ls gpurun_out/*.ncu-rep
