# A/B of alternative library builds on one config: gpu_libab.sh <cfg> lib1 lib2 ...
mkdir -p gpurun_out
cfg=$1; shift
for lib in "$@"; do
  SWX_LIB=$PWD/paper_1805_06557_b200/$lib timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$cfg $lib', 'ms/step %.4f'%d['ms_per_step'], {k: round(v['ms_per_launch']*1e3,1) for k,v in d['kernel_breakdown_ms'].items()})" || tail -3 gpurun_out/ab.err
done
