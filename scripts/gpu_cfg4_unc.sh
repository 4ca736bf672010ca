# cfg4 without the pivot cache over builds: bash scripts/gpu_cfg4_unc.sh <lib suffix>...
mkdir -p gpurun_out
for v in "$@"; do
  SWX_L_CACHE=0 SWX_LIB=$PWD/paper_1805_06557_b200/libswx_$v.so timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('uncached $v',round(d['ms_per_step'],3),'ms')"
done
