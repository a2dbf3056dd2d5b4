# usage: bash tools/ab_nch.sh ; x-chunk count sweep of star_tma at C1 (256^3) and 512^3 (SDMP_STAR_NCH)
run() { python bench.py --shape $1 --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 nch=$2', round(d['value'],1), round(d['roofline']['launch_ms']*1000,2), 'us', round(d['roofline']['frac'],3))"; }
for n in auto 2 3 4 5 6 7 8 10 12 16 24; do
  if [ $n = auto ]; then unset SDMP_STAR_NCH; else export SDMP_STAR_NCH=$n; fi
  run 256,256,256 $n
done
for n in auto 2 3 4 6 8; do
  if [ $n = auto ]; then unset SDMP_STAR_NCH; else export SDMP_STAR_NCH=$n; fi
  run 512,512,512 $n
done
