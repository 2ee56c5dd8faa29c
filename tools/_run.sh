set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
for v in default noval; do
if [ $v = default ]; then LP=""; else LP=$PWD/paper_2108_01731_b200/_lib/ab_$v/liblcc_b200.so; fi
for i in 1 2 3 4; do
LCC_LIB_PATH=$LP timeout 600 python bench.py --no-cpu --steps 3 --e2e-steps 1 > $O/b.json 2>/dev/null; python -c "import json;d=json.load(open('$O/b.json'));e=d['e2e'];print('$v', round(d['value'],2), d['round_stats']['moves'], 'e2e', round(e['value'],2), round(e['clustering_ms'],1), e['levels'], e['rounds'], round(e['objective']))"
done; done
