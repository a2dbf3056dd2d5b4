# usage: bash tools/ab_run.sh variant... ; per-variant family timings (512^3)
for v in "$@"; do
  for k in "tti 8" "elastic 8" "visco 16"; do set -- $k
  SDMP_LIB=abtest/libsdmp_$v.so python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', '$1', round(d['value'],2), [ (a['kind'], round(a['ms'],3)) for a in d['step_actions'] if a['ms']>0.05])"
  done
done
