for v in 0 7; do for so in 14 16; do
SDMP_STAR_VARIANT=$v python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('variant $v SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))"
done; done
bash tools/so_sweep.sh
