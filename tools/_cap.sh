# GPU tests + bench + one full ncu capture of the best-move kernels of one step;
# the report itself stays on the box (too large to merge back), CSV extracts come back.
set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench_new.json 2> $O/bench_new.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/launches_new.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $O/ncu_launch_new.log 2>&1
echo "launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_group|k_small|k_large_insert|k_large_score|k_large_mark|k_isolated|k_edge_balanced' -s 0 -c 40 \
  -o /tmp/full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $O/ncu_full_new.log 2>&1
echo "full rc=$?"
ncu -i /tmp/full.ncu-rep --page raw --csv > $O/full_raw.csv 2>/dev/null
for k in 'k_group<WNone, 1, 1, 1024' 'k_group<WNone, 1, 1, 256' 'k_small' 'k_large_insert'; do
  f=$(echo "$k" | tr -c 'a-zA-Z0-9' '_')
  ncu -i /tmp/full.ncu-rep --page source --csv --print-source cuda,sass -k "regex:$k" -c 1 > $O/src_$f.csv 2>/dev/null
done
ls -la /tmp/full.ncu-rep
