# one iteration: GPU parity tests, cfg2 bench, ncu launch list of the cfg2 step
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "relative L2|passed|failed|Error|error" gpurun_out/pytest_gpu.log | head -20
timeout 600 python bench.py --steps 48 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('ms/step %.4f'%d['ms_per_step'], 'value %.3e'%d['value'], 'roof', d['roofline'] and (d['roofline']['kernel'], round(d['roofline']['frac'] or 0,3)), 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],3))
print({k: round(v['ms_per_step']*1e3,1) for k,v in d['kernel_breakdown_ms'].items()})
"
CMD="python bench.py --steps 2 --warmup 1 --profile"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
