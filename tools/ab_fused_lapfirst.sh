# A/B: single-pass TTI with the Laplacian of p formed before the product-plane stores (tap loads reused)
out=gpurun_out/r5j_ab.txt; rm -f $out
for rep in 1 2; do for lib in product lf1 m4 lf1m4; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for so in 4 6 8; do
    timeout 300 python bench.py --kernel tti --so $so --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'tti', $so, round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
