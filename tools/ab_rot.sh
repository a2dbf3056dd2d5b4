# usage: bash tools/ab_rot.sh variant... ; rotated (tti_gxx_kernel) SO-4/8/16 per libsdmp variant (abtest/)
for v in "$@"; do for so in 4 8 16; do
SDMP_LIB=abtest/libsdmp_$v.so python bench.py --kernel rotated --so $so --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v rotated', $so, round(d['value'],2), round(d['roofline']['frac'],3), [(a['kind'], a['ms']) for a in d['step_actions'] if a['ms'] > 0.05])"
done; done
