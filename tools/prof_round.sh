#!/usr/bin/env bash
# Per-launch times and DRAM traffic of one bench step (round kernels only),
# for each config given; then profiles/TAG_traffic_CFG.json.
# Usage (GPU box): bash tools/prof_round.sh TAG cfg5 cfg4
set -u
T=$1; shift
O=gpurun_out; mkdir -p $O
K='regex:k_group|k_small|k_tiny|k_hub|k_isolated|k_large|k_bin|k_mass|k_relabel|k_min_member|k_pack|k_labels|k_degrees|DeviceCompact|DeviceSelect|DeviceScan'
for CFG in "$@"; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "$K" -c 300 --csv --log-file $O/${T}_${CFG}_launches.csv \
    python bench.py --config $CFG --extra-config none --steps 1 --warmup 0 --no-cpu --no-e2e > $O/${T}_${CFG}_launch.log 2>&1 \
    || echo "launch list $CFG failed"
  python tools/traffic_step.py $O/${T}_${CFG}_launches.csv $CFG $T
done
