# A/B: elastic velocity / stress with 2 resident CTAs per SM (more tiles in flight) vs 1, at the C4 per-GPU cross-sections
out=gpurun_out/r5f_ab.txt; rm -f $out
for rep in 1 2; do for lib in product sc2 vc2 svc2; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for shp in 1024,1024,1024 512,512,1024 512,512,512; do
    timeout 300 python bench.py --kernel elastic --so 8 --shape $shp --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'elastic SO-8 $shp', round(d['value'],2), round(d['roofline']['frac'],3), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
  done; done; done
unset SDMP_LIB
