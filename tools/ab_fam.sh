# usage: bash tools/ab_fam.sh variant... ; stream-engine families per libsdmp variant (abtest/)
for v in "$@"; do
  for k in "tti 4 512" "tti 8 512" "tti 16 512" "rotated 8 512" "elastic 8 512" "elastic 16 512" "visco 8 512" "visco 16 512" "damped 8 1024" "damped 16 1024"; do set -- $k
  SDMP_LIB=abtest/libsdmp_$v.so python bench.py --kernel $1 --so $2 --shape $3,$3,$3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$1', $2, round(d['value'],2), round(d['roofline']['frac'],3))"
  done
done
