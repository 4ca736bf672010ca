# cfg4 (T1279, N=1024) with / without the pivot cache, default and fast-reciprocal builds
mkdir -p gpurun_out
run() { # label, env...
  lbl=$1; shift
  env "$@" timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$lbl',round(d['ms_per_step'],3),'ms', d['run_info'].get('l_pivot_cache_bytes'))"
}
run "cached default" X=1
run "uncached default" SWX_L_CACHE=0
run "uncached fastrcp" SWX_L_CACHE=0 SWX_LIB=$PWD/paper_1805_06557_b200/libswx_frcp.so
run "cached fastrcp" SWX_LIB=$PWD/paper_1805_06557_b200/libswx_frcp.so
SWX_LIB=$PWD/paper_1805_06557_b200/libswx_frcp.so SWX_L_PART=0 python -m pytest tests -m gpu -x -q -k "l_ or cfg1 or cfg4 or chain or pole" 2>&1 | tail -2
