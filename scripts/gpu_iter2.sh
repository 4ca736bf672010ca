# parity tests + cfg2 bench + multi-rank code path on 1 GPU (torchrun, forced comm)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "relative L2|passed|failed|Error|error" gpurun_out/pytest_gpu.log | head -20
timeout 600 python bench.py --steps 48 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('ms/step %.4f'%d['ms_per_step'], 'value %.3e'%d['value'], 'roof', d['roofline'] and (d['roofline']['kernel'], round(d['roofline']['frac'] or 0,3)), 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],3))
print({k: round(v['ms_per_step']*1e3,1) for k,v in d['kernel_breakdown_ms'].items()})
"
for c in cfg2 cfg1; do
SWX_FORCE_COMM=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --config $c --steps 5 --warmup 2 > gpurun_out/bench_comm_$c.json 2> gpurun_out/bench_comm_$c.err; echo "torchrun forced-comm $c rc=$?"; tail -3 gpurun_out/bench_comm_$c.err | grep -v Warn; cut -c1-300 gpurun_out/bench_comm_$c.json
done
