mkdir -p gpurun_out
for cfg in cfg1 cfg4; do
  for lib in libswx.so libswx_seg8.so; do
    SWX_LIB=$PWD/paper_1805_06557_b200/$lib timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/lc.json 2> gpurun_out/lc.err
    python -c "
import json; d=json.load(open('gpurun_out/lc.json'))
print('$cfg $lib', 'ms/step %.4f'%d['ms_per_step'], 'value %.3e'%d['value'])" || tail -3 gpurun_out/lc.err
  done
done
SWX_LIB=$PWD/paper_1805_06557_b200/libswx_seg8.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "l_golden or t21 or t42 or cfg1 or cfg4 or pole or prepared or axpy or two_rhs or singular or stiff or split" 2>&1 | tail -3
