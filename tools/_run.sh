set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -15 $O/gpu_tests.log
LCC_BENCH_DEBUG=1 LCC_TRACE=1 timeout 600 python bench.py --no-cpu --steps 3 --e2e-steps 3 > $O/bench_dbg.json 2> $O/bench_dbg.err; echo "dbg rc=$?"
grep "e2e phases\|compress ->\|level\|unwind" $O/bench_dbg.err | tail -24
python -c "import json;d=json.load(open('$O/bench_dbg.json'));print(d['value'], d['e2e']['value'], d['e2e']['clustering_ms'])"
