# A/B: TTI update pass (R = 4) tile rows: 12 (product, 13 warps, 128-register cap), 11 (12 warps, 168), 7 (8 warps, 255)
out=gpurun_out/r2w_ab.txt; rm -f $out
for rep in 1 2; do for lib in product uty11 uty7; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  python bench.py --kernel tti --so 8 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), round(d['roofline']['frac'],3), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
done; done
unset SDMP_LIB
# visco SO-4/8 stress (NP = 15) and elastic velocity at 15-row tiles (16 warps, 128-register cap) vs 16 rows (17 warps, 96)
for rep in 1 2; do for lib in product ty15; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for ks in "visco 4" "visco 8" "elastic 8"; do set -- $ks
  python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, round(d['value'],1), round(d['roofline']['frac'],3), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
  done; done; done
unset SDMP_LIB
