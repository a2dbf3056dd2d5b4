# usage: bash tools/ab_ty8.sh ; star_tma 16-row (1 CTA/SM) vs 8-row (2 CTAs/SM, SDMP_STAR_VARIANT=8) tiles
run() { python bench.py --shape $1 --steps $2 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 v=${SDMP_STAR_VARIANT:-0} nch=${SDMP_STAR_NCH:-auto}', round(d['value'],1), round(d['roofline']['launch_ms']*1000,2), 'us', round(d['roofline']['frac'],3))"; }
for v in 0 8; do export SDMP_STAR_VARIANT=$v; unset SDMP_STAR_NCH
  run 256,256,256 200; run 512,512,512 100; run 1024,1024,1024 30
  if [ $v = 8 ]; then for n in 2 3 4 6 8; do export SDMP_STAR_NCH=$n; run 256,256,256 200; done; fi
done
