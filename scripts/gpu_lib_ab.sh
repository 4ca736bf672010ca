# cfg2 line over alternative builds: bash scripts/gpu_lib_ab.sh <lib suffix>...
mkdir -p gpurun_out
for v in "" "$@" "" "$@"; do
  lib=paper_1805_06557_b200/libswx${v:+_$v}.so
  SWX_LIB=$PWD/$lib python bench.py --steps 48 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('lib=$v', round(d['ms_per_step']*1e3,2),'us', {k: round(v['ms_per_launch']*1e3,1) for k,v in d['kernel_breakdown_ms'].items()})"
done
