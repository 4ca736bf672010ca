# cfg1 (and optionally cfg4) bench of the thread-per-chain kernel over pivot-ring depths
mkdir -p gpurun_out
for v in "" "$@"; do
  lib=paper_1805_06557_b200/libswx${v:+_$v}.so
  SWX_L_PART=0 SWX_LIB=$PWD/$lib python bench.py --config cfg1 --steps 20 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('cfg1 lib=$v',round(d['ms_per_step']*1e3,1),'us')"
done
SWX_L_PART=0 SWX_L_CACHE=0 python bench.py --config cfg1 --steps 20 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('cfg1 uncached',round(d['ms_per_step']*1e3,1),'us')"
