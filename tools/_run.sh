set -u
O=gpurun_out; mkdir -p $O
LCC_BENCH_DEBUG=1 LCC_TRACE=1 timeout 600 python bench.py --no-cpu --steps 3 --e2e-steps 3 > $O/bench_dbg.json 2> $O/bench_dbg.err; echo "dbg rc=$?"
grep "e2e\|compress keys" $O/bench_dbg.err | tail -20
