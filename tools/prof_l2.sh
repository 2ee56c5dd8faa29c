#!/usr/bin/env bash
# L2 / DRAM breakdown of the best-move kernels of one bench step (config 5
# by default): sectors by op and hit/miss, evict-class requests, fabric
# (cross-die) sectors, DRAM bytes.  Caches are NOT flushed between kernels
# (--cache-control none) so the numbers describe the live step.
# Usage: bash tools/prof_l2.sh TAG [cfg] [extra env assignments...]
set -u
T=${1:-r02}; CFG=${2:-cfg5}; shift 2 || true
O=gpurun_out; mkdir -p $O
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_requests_srcunit_tex_op_write.sum,lts__t_requests_srcunit_tex_op_atom.sum,lts__t_requests_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__d_sectors_fill_device.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_requests_srcunit_tex_evict_first.sum,lts__t_requests_srcunit_tex_evict_first_lookup_hit.sum,lts__t_requests_srcunit_tex_evict_last.sum,lts__t_requests_srcunit_tex_evict_last_lookup_hit.sum,lts__t_requests_srcunit_tex_evict_normal.sum,lts__t_requests_srcunit_tex_evict_normal_lookup_hit.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active
B="python bench.py --config $CFG --extra-config none --steps 1 --warmup 0 --no-cpu --no-e2e ${BENCH_EXTRA:-}"
env "$@" timeout 1200 ncu --metrics $M --cache-control none --clock-control none \
  -k 'regex:k_group|k_small|k_hub_bucket|k_hub_scatter|k_tiny' -c 120 --csv \
  --log-file $O/${T}_${CFG}_l2.csv $B > $O/${T}_${CFG}_l2.log 2>&1 || echo "l2 capture failed"
python tools/l2_summary.py $O/${T}_${CFG}_l2.csv > $O/${T}_${CFG}_l2.md 2>&1
