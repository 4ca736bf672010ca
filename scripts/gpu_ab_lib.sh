# A/B of two builds: libswx.so (A) vs libswx_alt.so (B), each with env variants
# usage: bash scripts/gpu_ab_lib.sh "ENV=a" "ENV=b" ...
mkdir -p gpurun_out
cp paper_1805_06557_b200/libswx.so /tmp/libA.so
for L in A B; do
  if [ $L = B ]; then cp paper_1805_06557_b200/libswx_alt.so paper_1805_06557_b200/libswx.so; fi
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$L.log 2>&1; echo "$L pytest: $(tail -1 gpurun_out/pytest_$L.log)"
  for V in "$@"; do
    env $V timeout 600 python bench.py --steps 48 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$L $V', 'ms/step %.4f'%d['ms_per_step'], {k: round(v['ms_per_step']*1e3,1) for k,v in d['kernel_breakdown_ms'].items()})"
  done
done
cp /tmp/libA.so paper_1805_06557_b200/libswx.so
