# A/B: single-pass TTI (ab/libsdmp_f4.so: fused up to R = 4) vs product (fused R <= 2)
out=gpurun_out/r2n_ab.txt; rm -f $out
for lib in product f4; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_f4.so; fi
  for so in 4 6 8; do for n in 512 768; do
    python bench.py --kernel tti --so $so --shape $n,$n,$n --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'SO-$so', $n, round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
