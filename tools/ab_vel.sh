# visco SO-16 / elastic SO-12 velocity: fused vs split (SDMP_VEL_SPLIT)
for sp in 0 1; do for k in "visco 16" "elastic 12"; do set -- $k
SDMP_VEL_SPLIT=$sp python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('split=$sp $1 SO-$2', round(d['value'],2), [(a['kind'], round(a['ms'],3)) for a in d['step_actions'] if a['ms']>0.05])"
done; done
