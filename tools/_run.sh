set -u
O=gpurun_out; mkdir -p $O
for i in 1 2 3 4 5; do
timeout 600 python bench.py --no-cpu --steps 3 --e2e-steps 3 > $O/b.json 2>/dev/null; python -c "import json;d=json.load(open('$O/b.json'));e=d['e2e'];print(round(d['value'],3), 'e2e', round(e['value'],2), round(e['clustering_ms'],1), round(e['device_ms_parallel_cc'],1), e['levels'], e['rounds'], round(e['objective']))"
done
