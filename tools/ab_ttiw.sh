# usage: bash tools/ab_ttiw.sh variant... ; TTI SO-12/16 per libsdmp variant (abtest/)
for v in "$@"; do for so in 12 16; do
SDMP_LIB=abtest/libsdmp_$v.so python bench.py --kernel tti --so $so --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v tti', $so, round(d['value'],2), round(d['roofline']['frac'],3))"
done; done
