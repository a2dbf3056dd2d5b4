# acoustic SO sweep at 1024^3 on one GPU (roofline per SO)
for so in 4 8 12 16; do
python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('SO-$so', round(d['value'],1), 'frac', round(r['frac'],3), r['kernel'], 'e2e', round(d['e2e']['value'],1))"
done
