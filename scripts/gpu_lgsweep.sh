mkdir -p gpurun_out
for cfgv in "8 8" "4 8" "2 8" "8 4" "4 16" "16 8" "8 16" "32 4"; do
  set -- $cfgv
  SWX_LG_LPM=$1 SWX_LG_LEAF=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); b=d['kernel_breakdown_ms']
print('lpm $1 leaf $2', 'step %.4f'%d['ms_per_step'], 'pair %.1f single %.1f'%(b['rexi_lg_pair']['ms_per_launch']*1e3, b['rexi_lg_single']['ms_per_launch']*1e3))
"
done
