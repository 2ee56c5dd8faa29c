set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu > $O/b.json 2>/dev/null; python -c "import json;d=json.load(open('$O/b.json'));e=d['e2e'];print(round(d['value'],2), 'e2e', round(e['value'],2), round(e['clustering_ms'],1), e['clustering_ms_per_step'], e['levels'], e['rounds'], round(e['objective']))"
done
