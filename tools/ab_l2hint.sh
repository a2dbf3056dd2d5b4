# A/B: stream-engine L2 hints (hint: fronts / centres evict_last, pointwise evict_first),
# streaming .cs output stores (cs), both (hintcs) vs product; 512^3 and 1024^3
out=gpurun_out/r3l_ab.txt; rm -f $out
for lib in product hint cs hintcs; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for ks in "elastic 8 1024" "elastic 8 512" "visco 8 512" "damped 8 1024" "tti 8 512"; do set -- $ks
  python bench.py --kernel $1 --so $2 --shape $3,$3,$3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, $3, round(d['value'],2), round(d['roofline']['frac'],3), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
  done; done
unset SDMP_LIB
