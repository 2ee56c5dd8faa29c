set -u
O=gpurun_out; mkdir -p $O
for r in 1 2; do
  timeout 300 python bench.py --no-cpu --no-e2e > $O/ab_pipe1_$r.json 2>/dev/null
  LCC_LIB_PATH=$PWD/paper_2108_01731_b200/_lib/ab0/liblcc_b200.so timeout 300 python bench.py --no-cpu --no-e2e > $O/ab_pipe0_$r.json 2>/dev/null
done
LCC_BENCH_DEBUG=1 LCC_TRACE=1 timeout 600 python bench.py --no-cpu --steps 3 > $O/bench_dbg.json 2> $O/bench_dbg.err; echo "dbg rc=$?"
for f in $O/ab_*.json; do echo $f $(python -c "import json;print(json.load(open('$f'))['value'])"); done
