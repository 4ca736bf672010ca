mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "relative L2|passed|failed|Error|error" gpurun_out/pytest_gpu.log | head -20
for c in cfg1 cfg4 cfg0; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
  tail -2 gpurun_out/bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json'))
print('$c', 'ms/step %.4f'%d['ms_per_step'], 'value %.3e'%d['value'], 'roof', d['roofline'] and (d['roofline']['kernel'], round(d['roofline']['frac'] or 0,3)), 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],3))
"
done
