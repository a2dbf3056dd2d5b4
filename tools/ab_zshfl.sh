# A/B: z neighbourhood by warp shuffles (ab/libsdmp_zshfl.so) vs staged-row loads (product)
out=gpurun_out/r2s_ab.txt; rm -f $out
for rep in 1 2; do for lib in product zshfl; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_zshfl.so; fi
  for so in 4 8 12 16; do
    python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
for lib in product zshfl; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_zshfl.so; fi
  SDMP_STAR_VARIANT=3 python bench.py --kernel acoustic --so 16 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib star_tma<8> (variant 3)', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
done
unset SDMP_LIB
