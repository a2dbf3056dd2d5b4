# A/B: staggered velocity with two y rows per thread (stream-engine kRows = 2; y taps shared)
# at 8 / 14-row tiles vs one row (product)
out=gpurun_out/r5b_ab.txt; rm -f $out
for rep in 1 2; do for lib in product r2t8 r2t14; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for k in "elastic 16" "elastic 12" "visco 16" "elastic 8"; do set -- $k
    timeout 300 python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, round(d['value'],2), round(d['roofline']['frac'],3), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
  done; done; done
unset SDMP_LIB
