# A/B: wide velocity launch shapes (z points per thread V, tile rows) vs product (V = 2, 8 rows)
out=gpurun_out/r4l_ab.txt; rm -f $out
for rep in 1 2; do for lib in product v1t16 v1t12 v2t12 v2t10; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for k in "elastic 16" "elastic 12"; do set -- $k
    timeout 300 python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, round(d['value'],2), round(d['roofline']['frac'],3), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
  done; done; done
unset SDMP_LIB
