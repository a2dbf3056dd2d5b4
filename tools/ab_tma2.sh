# usage: bash tools/ab_tma2.sh variant... ; acoustic SO-12/14/16 (star_tma2) per libsdmp variant
for v in "$@"; do for so in 12 14 16; do
SDMP_LIB=abtest/libsdmp_$v.so python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))"
done; done
