# A/B: single-pass TTI / rotated with decoupled product-plane barriers (halo roles run a plane ahead)
out=gpurun_out/r5i_ab.txt; rm -f $out
for rep in 1 2; do for lib in product sb1 m4 sb1m4; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for k in "tti 4" "tti 6" "tti 8" "rotated 4" "rotated 6" "rotated 8"; do set -- $k
    [ $1 = rotated ] && { [ $lib = m4 ] || [ $lib = sb1m4 ]; } && continue
    timeout 300 python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
