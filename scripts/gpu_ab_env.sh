# A/B of an environment knob on the cfg2 bench: usage gpu_ab_env.sh VAR "v1 v2 ..." [reps]
mkdir -p gpurun_out
VAR=$1; VALS=$2; REPS=${3:-2}
for r in $(seq $REPS); do
  for v in $VALS; do
    env $VAR=$v timeout 300 python bench.py --steps 48 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$VAR=$v', 'ms/step %.4f'%d['ms_per_step'], {k: round(v['ms_per_launch']*1e3,1) for k,v in d['kernel_breakdown_ms'].items()})"
  done
done
