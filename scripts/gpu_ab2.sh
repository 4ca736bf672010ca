# quick A/B of an env knob on the cfg2 bench: gpu_ab2.sh "label:ENV=V ENV2=V2" ...
mkdir -p gpurun_out
for r in 1 2; do
for spec in "$@"; do
  label=${spec%%:*}; envs=${spec#*:}
  env $envs timeout 300 python bench.py --steps 48 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$label', 'ms/step %.4f'%d['ms_per_step'], {k: round(v['ms_per_launch']*1e3,1) for k,v in d['kernel_breakdown_ms'].items()})" 2>/dev/null || tail -3 gpurun_out/ab.err
done
done
