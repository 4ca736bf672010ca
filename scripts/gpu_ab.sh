# A/B of env variants on the cfg2 bench: bash scripts/gpu_ab.sh "VAR=a" "VAR=b" ...
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for V in "$@"; do
  env $V timeout 600 python bench.py --steps 48 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$V', 'ms/step %.4f'%d['ms_per_step'], {k: round(v['ms_per_step']*1e3,1) for k,v in d['kernel_breakdown_ms'].items()})"
done
