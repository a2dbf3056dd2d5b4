set -e
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for k in "tti 8" "elastic 8" "visco 16"; do set -- $k
python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['value'],2), d['ms_per_step'], d['roofline']['frac'], d['clocks'], [ (a['kind'], a['ms']) for a in d['step_actions'] if a['ms']>0.05])"
done
