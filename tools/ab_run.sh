# Run bench.py (round only) for each ab_* variant and the default, alternating.
# Usage: bash tools/ab_run.sh REPS [extra bench args]
set -u
REPS=${1:-2}; shift || true
O=gpurun_out; mkdir -p $O
for r in $(seq $REPS); do
  timeout 300 python bench.py --no-cpu --no-e2e "$@" > $O/ab_default_$r.json 2>/dev/null
  for d in paper_2108_01731_b200/_lib/ab_*; do
    n=$(basename $d)
    LCC_LIB_PATH=$PWD/$d/liblcc_b200.so timeout 300 python bench.py --no-cpu --no-e2e "$@" > $O/${n}_$r.json 2>/dev/null
  done
done
for f in $O/ab_*.json; do echo $f $(python -c "import json;d=json.load(open('$f'));x=d.get('cfg4') or {};print(round(d['value'],3), round(d['roofline']['kernel_ms_per_step'],3), round(x.get('value',0),3), round((x.get('roofline') or {}).get('kernel_ms_per_step',0),3))" 2>/dev/null); done
