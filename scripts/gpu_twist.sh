mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "l_golden or t21 or t42 or cfg1 or cfg4 or pole or prepared or axpy or two_rhs or split or singular or l_rexi_n" 2>&1 | tail -4
for cfg in cfg1 cfg4; do
  for t in 0 1; do
    SWX_L_TWIST=$t timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/lc.json 2> gpurun_out/lc.err
    python -c "
import json; d=json.load(open('gpurun_out/lc.json'))
print('$cfg SWX_L_TWIST=$t', 'ms/step %.4f'%d['ms_per_step'])" || tail -3 gpurun_out/lc.err
  done
done
