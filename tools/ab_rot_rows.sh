# A/B: single-pass rotated operator with 16-row tiles (g halo factor 1.69 instead of 2.25 at R = 4)
out=gpurun_out/r4w_ab.txt; rm -f $out
for rep in 1 2; do for lib in product rot16 rot16m6; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for so in 4 6 8 10 12; do
    timeout 300 python bench.py --kernel rotated --so $so --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'rotated SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
