# A/B of run-time knobs (env assignments) on the bench round, alternating.
# Usage: bash tools/ab_env.sh REPS "ENV=1" "ENV=0" ...
set -u
REPS=$1; shift
O=gpurun_out; mkdir -p $O
for r in $(seq $REPS); do
  i=0
  for e in "$@"; do
    env $e timeout 300 python bench.py --no-cpu --no-e2e > $O/abenv_${i}_$r.json 2>/dev/null
    echo "$e rep $r: $(python -c "import json;d=json.load(open('$O/abenv_${i}_$r.json'));x=d.get('cfg4') or {};print(round(d['value'],3), round(d['roofline']['kernel_ms_per_step'],3), round(x.get('value',0),3), round((x.get('roofline') or {}).get('kernel_ms_per_step',0),3))" 2>/dev/null)"
    i=$((i+1))
  done
done
