# A/B: star_tmem launch shapes (rows per CTA, x-tap batch, pipeline stages) at acoustic SO-14/16
out=gpurun_out/r4d_ab.txt; rm -f $out
for rep in 1 2; do for lib in product rows20 rows28 rows20kc8 st5; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for so in 14 16; do
    timeout 120 python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
