# full ncu capture of selected kernels of the cfg2 step: bash scripts/gpu_ncu.sh regex1 regex2 ...
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --profile"
for K in "$@"; do
  $CMD > gpurun_out/plain_$K.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1
  echo "$K rc=$?"
done
