mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --profile"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
for K in analysis_kernel synth_state_kernel rexi_lg_kernel; do
  $CMD > gpurun_out/plain_$K.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1
  echo "$K rc=$?"
done
ls -la gpurun_out
