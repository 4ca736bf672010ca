# cfg2 / cfg0 / cfg3 quick A/B after an lg kernel change: tests touching lg + bench lines
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "lg or cfg0 or etdrk or fused or prepared or handoff or race or pole or cfg3" > gpurun_out/lg_tests.log 2>&1; tail -2 gpurun_out/lg_tests.log
for c in cfg2 cfg0; do
python bench.py --config $c --steps 48 --no-cpu --no-e2e > gpurun_out/ab_$c.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab_$c.json'));print('$c', round(d['ms_per_step']*1e3,2),'us', {k: round(v['ms_per_launch']*1e3,1) for k,v in d['kernel_breakdown_ms'].items()})"
done
