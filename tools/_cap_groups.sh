set -u
O=gpurun_out; mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_group|k_small' -s 0 -c 6 \
  -o /tmp/g python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $O/ncu_g.log 2>&1 || echo "capture failed"
ncu -i /tmp/g.ncu-rep --page raw --csv > $O/g_raw.csv 2>/dev/null
for i in 0 1 2 3 4 5; do
  ncu -i /tmp/g.ncu-rep --page source --csv --print-source cuda,sass -s $i -c 1 > $O/g_src_$i.csv 2>/dev/null
done
ls -la $O
