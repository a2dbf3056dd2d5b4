# usage: bash tools/ab_tti.sh variant... ; TTI SO-8 (and rotated SO-8) per libsdmp variant (abtest/)
for v in "$@"; do for k in "tti 8" "rotated 8"; do set -- $k
SDMP_LIB=abtest/libsdmp_$v.so python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$1', $2, round(d['value'],2), round(d['roofline']['frac'],3))"
done; done
