# A/B: component-split velocity op (VelSplitOpT: one warp group per velocity component, 2 rows
# per thread; product from SO-10) vs the all-components op (ab/libsdmp_nosplit.so); tile heights
out=gpurun_out/r4g_ab.txt; rm -f $out
for rep in 1 2; do for lib in product nosplit ty10 ty6 split3; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for k in "elastic 16" "visco 16" "elastic 12" "elastic 8" "elastic_col 8"; do set -- $k
    [ $lib = split3 ] || [ $2 -ge 10 ] || continue
    timeout 300 python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, round(d['value'],2), round(d['roofline']['frac'],3), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
  done; done; done
unset SDMP_LIB
