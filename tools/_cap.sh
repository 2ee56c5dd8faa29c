set -u
O=gpurun_out; mkdir -p $O
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_group|k_small|k_isolated' -s 0 -c 7 \
  -o /tmp/grp python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > $O/ncu_grp.log 2>&1
echo "full rc=$?"
ncu -i /tmp/grp.ncu-rep --page raw --csv > $O/grp_raw.csv 2>/dev/null
for i in 0 1 2 3 4 5 6; do
  ncu -i /tmp/grp.ncu-rep --page source --csv --print-source cuda,sass -s $i -c 1 > $O/grp_src_$i.csv 2>$O/grp_src_$i.err
done
ls -la /tmp/grp.ncu-rep; cp /tmp/grp.ncu-rep $O/ 2>/dev/null; du -sh $O
