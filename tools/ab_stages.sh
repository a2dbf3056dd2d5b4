# A/B: star_tma / star_tma2 pipeline depth 4 (product) vs 5 / 6 stages
out=gpurun_out/r3c_ab.txt; rm -f $out
for rep in 1 2; do for lib in product s5 s6; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for so in 8 12 16; do
  python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
