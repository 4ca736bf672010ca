# cfg2 step A/B after a kernel change: the whole GPU suite + the cfg2 line
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
for i in 1 2; do
python bench.py --steps 48 --no-cpu --no-e2e > gpurun_out/ab_cfg2.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab_cfg2.json'));print('cfg2', round(d['ms_per_step']*1e3,2),'us', {k: round(v['ms_per_launch']*1e3,1) for k,v in d['kernel_breakdown_ms'].items()})"
done
