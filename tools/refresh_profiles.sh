#!/usr/bin/env bash
# Regenerate the round's measurement evidence on a GPU box (run under gpurun):
#   bench line (ours + reference arm), the ncu launch list of the bench
#   command, and `ncu --set full` captures of the best-move kernels of one
#   step (warp/CTA groups + small bin in one report, the hub path in another).
#   Reports stay on the box (too large to merge back); raw-metric and
#   source-view CSV extracts come back in gpurun_out/.
# Usage: bash tools/refresh_profiles.sh RND [captures]   (captures: skip the bench lines)
set -u
R=${1:-01}
O=gpurun_out
mkdir -p $O
if [ "${2:-}" != "captures" ]; then
timeout 600 python bench.py > $O/bench_r$R.json 2> $O/bench_r$R.err || { echo "bench failed"; tail -5 $O/bench_r$R.err; exit 1; }
timeout 600 python bench.py --impl reference > $O/bench_ref_r$R.json 2> $O/bench_ref_r$R.err || echo "reference arm failed"
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file $O/launches_r$R.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $O/ncu_launch_r$R.log 2>&1 \
  || echo "launch list failed"
timeout 1200 ncu --set full -f --clock-control none --import-source on \
  -k 'regex:k_group|k_small|k_tiny|k_isolated' -s 0 -c 8 \
  -o /tmp/r${R}_groups python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $O/ncu_groups_r$R.log 2>&1 \
  || echo "groups capture failed"
timeout 1200 ncu --set full -f --clock-control none --import-source on \
  -k 'regex:k_hub|k_large' -s 0 -c 4 \
  -o /tmp/r${R}_hubs python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $O/ncu_hubs_r$R.log 2>&1 \
  || echo "hub capture failed"
for rep in groups hubs; do
  ncu -i /tmp/r${R}_$rep.ncu-rep --page raw --csv > $O/r${R}_${rep}_raw.csv 2>/dev/null
done
for i in 0 1 2 3 4 5 6 7; do
  ncu -i /tmp/r${R}_groups.ncu-rep --page source --csv --print-source cuda,sass -s $i -c 1 > $O/r${R}_groups_src_$i.csv 2>/dev/null
done
for i in 0 1; do
  ncu -i /tmp/r${R}_hubs.ncu-rep --page source --csv --print-source cuda,sass -s $i -c 1 > $O/r${R}_hubs_src_$i.csv 2>/dev/null
done
echo done
