# partition-kernel check: l-group parity tests, smoke, cfg1 bench with and without it
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "l_ or cfg1 or chain or pole or rexi or etdrk or strang or race or smoke" > gpurun_out/lpart_tests.log 2>&1; tail -5 gpurun_out/lpart_tests.log
python __graft_entry__.py 2>&1 | tail -2
for v in 1 0; do
  SWX_L_PART=$v python bench.py --config cfg1 --steps 20 > gpurun_out/bench_cfg1_part$v.json 2> gpurun_out/bench_cfg1_part$v.err
  python -c "import json;d=json.load(open('gpurun_out/bench_cfg1_part$v.json'));print('part=$v',d['ms_per_step'],d['kernel_breakdown_ms'],d['e2e']['ms_per_step'])" || tail -5 gpurun_out/bench_cfg1_part$v.err
done
