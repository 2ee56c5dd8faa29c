#!/usr/bin/env bash
# Round-2 evidence for the headline (config 5) step, on a GPU box under gpurun:
#   the ncu launch list of one bench step (round kernels only), and an
#   `ncu --set full` capture of the best-move kernels of that step (raw and
#   source CSV extracts come back in gpurun_out/).
# Usage: bash tools/prof_cfg5.sh TAG [cfg]
set -u
T=${1:-r02}; CFG=${2:-cfg5}
O=gpurun_out; mkdir -p $O
K='regex:k_group|k_small|k_tiny|k_hub|k_isolated|k_large|k_bin|k_mass|k_relabel|k_min_member|k_pack|k_degrees|DeviceCompact|DeviceSelect|DeviceScan'
B="python bench.py --config $CFG --extra-config none --steps 1 --warmup 0 --no-cpu --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 200 --csv \
  --log-file $O/${T}_${CFG}_launches.csv $B > $O/${T}_${CFG}_launch.log 2>&1 || echo "launch list failed"
timeout 1500 ncu --set full -f --clock-control none --import-source on \
  -k 'regex:k_group|k_small|k_tiny|k_hub_bucket|k_hub_scatter' -c 10 \
  -o /tmp/${T}_${CFG}_full $B > $O/${T}_${CFG}_full.log 2>&1 || echo "full capture failed"
ncu -i /tmp/${T}_${CFG}_full.ncu-rep --page raw --csv > $O/${T}_${CFG}_full_raw.csv 2>/dev/null
for i in 0 1 2 3 4 5 6 7 8 9; do
  ncu -i /tmp/${T}_${CFG}_full.ncu-rep --page source --csv --print-source cuda,sass -s $i -c 1 > $O/${T}_${CFG}_src_$i.csv 2>/dev/null
done
ls -la $O/${T}_${CFG}_* | head -20
