# bench lines of every config into gpurun_out/bench_<cfg>.json
mkdir -p gpurun_out
for cfg in cfg0 cfg1 cfg4 cfg2; do
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-20} --warmup 3 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$?"; tail -c 400 gpurun_out/bench_$cfg.err | tail -2
done
