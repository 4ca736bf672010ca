# cfg1 bench over builds of the partition kernel: bash scripts/gpu_lpart_ab.sh <lib suffix>...
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "l_ or cfg1 or chain or pole or rexi" > gpurun_out/lpart_tests.log 2>&1; tail -2 gpurun_out/lpart_tests.log
for v in "" "$@"; do
  lib=paper_1805_06557_b200/libswx${v:+_$v}.so
  SWX_LIB=$PWD/$lib python bench.py --config cfg1 --steps 20 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('lib=$v',round(d['ms_per_step']*1e3,1),'us')"
done
SWX_L_PART=0 python bench.py --config cfg1 --steps 20 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('thread-per-chain',round(d['ms_per_step']*1e3,1),'us')"
