# A/B: star_tmem shapes after the front-tile L2 hint (rows 28, x-tap batch 2, 3 stages) at SO-14/16
out=gpurun_out/r4v_ab.txt; rm -f $out
for rep in 1 2; do for lib in product rows28 kc2 st3; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for so in 14 16; do
    timeout 120 python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
