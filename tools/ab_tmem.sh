# A/B: acoustic SO-12/14/16 with the x-window in tensor memory (star_tmem, product at SO-16)
# vs the register-window star_tma2 (ab/libsdmp_reg.so) and launch-shape variants
out=gpurun_out/r4a_ab.txt; rm -f $out
for rep in 1 2; do for lib in product reg kc2 kc8 rows16 rows32 minr6; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for so in 12 14 16; do
    [ $so != 16 ] && [ $lib != minr6 ] && [ $lib != product ] && continue
    timeout 120 python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
