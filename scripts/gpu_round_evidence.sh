# round-end evidence (r02): bench lines of every config, the cfg2 launch list,
# ncu --set full of the dominant kernels, and the per-CTA trace of one cfg2
# step -> gpurun_out/
mkdir -p gpurun_out
for cfg in cfg0 cfg1 cfg4 etd1279 cfg3 cfg2; do
  timeout 1200 python bench.py --config $cfg --steps ${STEPS:-20} --warmup 3 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$?"; tail -c 300 gpurun_out/bench_$cfg.err | tail -1
done
# the multi-rank code paths at one rank (pole shards with the tree reduce; column shards over NCCL)
SWX_FORCE_COMM=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --shard poles --steps 10 --no-cpu > gpurun_out/bench_cfg2_forced_comm.json 2> gpurun_out/bench_cfg2_forced_comm.err; echo "forced comm poles rc=$?"
SWX_FORCE_COMM=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --shard cols --steps 10 --no-cpu > gpurun_out/bench_cfg2_cols_k1_nccl.json 2> gpurun_out/bench_cfg2_cols_k1_nccl.err; echo "forced comm cols rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --profile"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
for K in synth_ws grid_sq1 analysis_tab rexi_lg_mm; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1; echo "$K rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:rexi_l_part_kernel -s 1 -c 1 -o gpurun_out/prof_rexi_l_part_cfg1 python bench.py --config cfg1 --steps 1 --warmup 1 --profile > gpurun_out/ncu_l1.log 2>&1; echo "l part cfg1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:rexi_l_kernel -s 1 -c 1 -o gpurun_out/prof_rexi_l_cfg4 python bench.py --config cfg4 --steps 1 --warmup 1 --profile --no-cpu --no-e2e > gpurun_out/ncu_l4.log 2>&1; echo "l cfg4 rc=$?"
if [ -f paper_1805_06557_b200/libswx_trace.so ]; then
  SWX_LIB=$PWD/paper_1805_06557_b200/libswx_trace.so SWX_TRACE_OUT=gpurun_out/trace_step_cfg2.npy timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "trace rc=$?"
fi
for f in gpurun_out/prof_*.ncu-rep; do python scripts/ncu_metrics.py $f > ${f%.ncu-rep}_raw.txt 2>&1; done
ls gpurun_out/*.ncu-rep
