# A/B: single-pass rotated operator up to R = 4 (ab/libsdmp_r4.so) vs product (R <= 2)
out=gpurun_out/r2p_ab.txt; rm -f $out
for lib in product r4; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_r4.so; fi
  for so in 4 6 8; do
    python bench.py --kernel rotated --so $so --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done
unset SDMP_LIB
