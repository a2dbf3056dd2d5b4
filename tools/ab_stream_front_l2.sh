# A/B: stream-engine front tiles loaded evict_last (ab/libsdmp_sfl2.so) vs product
out=gpurun_out/r4j_ab.txt; rm -f $out
for rep in 1 2; do for lib in product sfl2; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for k in "damped 8 1024" "damped 16 1024" "elastic 8 512" "elastic 16 512" "elastic 8 1024" "visco 16 512" "tti 8 512" "tti 16 512" "rotated 16 512"; do set -- $k
    timeout 300 python bench.py --kernel $1 --so $2 --shape $3,$3,$3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, $3, round(d['value'],2), round(d['roofline']['frac'],3), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
  done; done; done
unset SDMP_LIB
