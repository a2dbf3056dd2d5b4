# A/B: star_tma segmented work split (end-to-end tile-planes per CTA, no wave tail) vs x chunks
out=gpurun_out/r5c_ab.txt; rm -f $out
for rep in 1 2; do for lib in product seg2 seg1; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  timeout 300 python bench.py --shape 256,256,256 --steps 200 --warmup 5 --mode diagonal --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'C1 256^3 SO-8', round(d['value'],1), round(d['roofline']['frac'],3), d['roofline']['launch_ms'])" >> $out
  for so in 4 8; do for n in 512 1024; do
    timeout 300 python bench.py --so $so --n $n --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'SO-$so ${n}^3', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done; done
unset SDMP_LIB
