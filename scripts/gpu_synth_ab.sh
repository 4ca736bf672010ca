# A/B of state-synthesis scheduling variants on the cfg2 bench
mkdir -p gpurun_out
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --steps 48 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$label', 'ms/step %.4f'%d['ms_per_step'], {k: round(v['ms_per_launch']*1e3,1) for k,v in d['kernel_breakdown_ms'].items()})" || tail -3 gpurun_out/ab.err
}
L2=$PWD/paper_1805_06557_b200/libswx_minb2.so
for r in 1 2; do
run default X=0
run items SWX_SYNTH_ITEMS=1
run minb2 SWX_LIB=$L2
run minb2+items SWX_LIB=$L2 SWX_SYNTH_ITEMS=1
run two+items SWX_SYNTH_TWO=1 SWX_SYNTH_ITEMS=1
done
