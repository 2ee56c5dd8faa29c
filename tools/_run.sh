set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
timeout 300 python bench.py --no-cpu --no-e2e > $O/b.json 2>/dev/null; python -c "import json;d=json.load(open('$O/b.json'));print(round(d['value'],3))"
