for v in "$@"; do
for k in "elastic 8 --shape 512,512,512" "elastic 4 --shape 512,512,512" "damped 8" "damped 4"; do set -- $k
SDMP_LIB=abtest/libsdmp_$v.so python bench.py --kernel $1 --so $2 $3 $4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $1 SO-$2', round(d['value'],2), [(a['kind'], round(a['ms'],3)) for a in d['step_actions'] if a['ms']>0.05])"
done; done
