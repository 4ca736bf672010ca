# One compute-sanitizer tool per gpurun call (memcheck | racecheck | synccheck | initcheck):
#   gpurun --timeout 1500 -- 'bash scripts/gpu_sanitize.sh memcheck'
# Covers smoke(), small ETD2RK steps (table analysis TMA/mbarrier ring, fused grid stage,
# PDL chain inside a CUDA graph), the l pole sum with the pivot cache (bulk-copy ring),
# the pole-block tree combine, and the column-sharded peer-store / direct-push paths
# (virtual ranks on one GPU).  Output: gpurun_out/sanitize_<tool>.txt
tool=${1:-memcheck}
mkdir -p gpurun_out
out=gpurun_out/sanitize_${tool}.txt
CS=/usr/local/cuda/bin/compute-sanitizer
extra=""
[ "$tool" = "memcheck" ] && extra="--leak-check no"
[ "$tool" = "racecheck" ] && extra="--racecheck-report all"
tests="test_cfg0_lg_rexi_golden or test_t42_l_golden or test_cfg1_l_rexi_golden or test_etdrk_t42_golden \
or test_tendency_t63_golden or test_pole_blocks_combine_bitwise or test_fused_axpy_sum_bitwise \
or test_column_sharded_tendency_peer_stores_bitwise or test_column_sharded_tendency_direct_push_bitwise \
or test_table_free_transforms_and_tendency_vs_oracle or test_singular_shifts_raise"
{
  echo "== $tool: smoke()"
  timeout 1200 $CS --tool $tool $extra --error-exitcode 97 --print-limit 50 python __graft_entry__.py
  echo "rc=$?"
  echo "== $tool: GPU parity subset"
  timeout 1200 $CS --tool $tool $extra --error-exitcode 97 --print-limit 50 \
    python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$tests"
  echo "rc=$?"
} > $out 2>&1
grep -E "ERROR SUMMARY|rc=|passed|failed|==" $out | tail -20
