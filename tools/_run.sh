set -u
O=gpurun_out; mkdir -p $O
for c in cfg1 cfg2 cfg3 cfg5; do
  LCC_TRACE=1 timeout 900 python bench.py --config $c --no-cpu > $O/bc_$c.json 2> $O/bc_$c.err; echo "$c rc=$?"
  python -c "import json;d=json.load(open('$O/bc_$c.json'));e=d['e2e'];print('$c', round(d['value'],2), round(d['ms_per_step'],2), 'e2e', round(e['value'],2), round(e['clustering_ms'],1), e['levels'], e['rounds'], e['objective'])" 2>&1 | tail -1
  grep "level\|compress ->\|unwind" $O/bc_$c.err | tail -12
done
