# A/B: star_tma / star_tma2 front tiles loaded evict_last (ab/libsdmp_tmal2.so) vs product, acoustic 1024^3
out=gpurun_out/r4i_ab.txt; rm -f $out
for rep in 1 2 3; do for lib in product tmal2; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for so in 4 8 12; do
    timeout 120 python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
