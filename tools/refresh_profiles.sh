#!/usr/bin/env bash
# Regenerate the round's measurement evidence on a GPU box (run under gpurun):
#   bench line (ours + reference arm), the ncu launch list of the bench
#   command, and one `ncu --set full` capture of the best-move kernels.
# Usage: bash tools/refresh_profiles.sh RND      (outputs in gpurun_out/)
set -u
R=${1:-01}
O=gpurun_out
mkdir -p $O
timeout 600 python bench.py > $O/bench_r$R.json 2> $O/bench_r$R.err || { echo "bench failed"; tail -5 $O/bench_r$R.err; exit 1; }
timeout 600 python bench.py --impl reference > $O/bench_ref_r$R.json 2> $O/bench_ref_r$R.err || echo "reference arm failed"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/launches_r$R.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $O/ncu_launch_r$R.log 2>&1 \
  || echo "launch list failed"
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_group|k_small|k_large_insert|k_large_score|k_isolated|k_edge_balanced' -s 0 -c 12 \
  -o $O/r${R}_full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $O/ncu_full_r$R.log 2>&1 \
  || echo "full capture failed"
echo done
