for v in "$@"; do for so in 8 16; do
SDMP_LIB=abtest/libsdmp_$v.so python bench.py --kernel visco --so $so --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v SO-$so', round(d['value'],2), [(a['kind'], round(a['ms'],3)) for a in d['step_actions'] if a['ms']>0.05])"
done; done
