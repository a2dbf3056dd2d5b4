# A/B: TTI g pass with two rows per thread (ab/libsdmp_g2.so) vs one (product)
out=gpurun_out/r2z_ab.txt; rm -f $out
for rep in 1 2; do for lib in product g2; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for so in 8 12 16; do
  python bench.py --kernel tti --so $so --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'tti', $so, round(d['value'],1), round(d['roofline']['frac'],3), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
  done; done; done
unset SDMP_LIB
