# usage: bash scripts/gpu_ncu_cfg.sh <config> <kernel-regex> [skip]
mkdir -p gpurun_out
CMD="python bench.py --config $1 --steps 1 --warmup 1 --profile"
$CMD > gpurun_out/plain_$1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$2 -s ${3:-1} -c 1 -o gpurun_out/prof_$1_$2 $CMD > gpurun_out/ncu_$1_$2.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_$1_$2.log
