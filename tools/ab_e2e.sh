# A/B of run-time knobs on the end-to-end clustering (bench e2e leg):
# clustering ms per call and the objective.  Usage: bash tools/ab_e2e.sh REPS "ENV=1" ...
set -u
REPS=$1; shift
O=gpurun_out; mkdir -p $O
for r in $(seq $REPS); do
  i=0
  for e in "$@"; do
    env $e timeout 400 python bench.py --no-cpu --steps 2 --warmup 1 --e2e-steps 4 > $O/abe2e_${i}_$r.json 2>/dev/null
    echo "$e rep $r: $(python -c "import json;d=json.load(open('$O/abe2e_${i}_$r.json'))['e2e'];print(d['clustering_ms_per_step'], d['objective'], d['rounds'], round(d['value'],2))" 2>/dev/null)"
    i=$((i+1))
  done
done
