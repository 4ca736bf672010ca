# cfg1 / cfg4 l-chain pole sums with and without the pivot cache + parity tests
mkdir -p gpurun_out
for cfg in cfg1 cfg4; do
  for c in 0 1; do
    SWX_L_CACHE=$c timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/lc.json 2> gpurun_out/lc.err
    python -c "
import json; d=json.load(open('gpurun_out/lc.json'))
print('$cfg SWX_L_CACHE=$c', 'ms/step %.4f'%d['ms_per_step'], 'value %.3e'%d['value'])" || tail -3 gpurun_out/lc.err
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "l_golden or t21 or t42 or cfg1 or cfg4 or pole or prepared or axpy or two_rhs or singular or stiff or split" 2>&1 | tail -3
