# A/B: single-pass TTI / rotated fronts loaded evict_last (ab/libsdmp_ffl2.so) vs product
out=gpurun_out/r4k_ab.txt; rm -f $out
for rep in 1 2; do for lib in product ffl2; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for k in "tti 4" "tti 6" "rotated 4" "rotated 6" "rotated 8"; do set -- $k
    timeout 300 python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, round(d['value'],2), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
