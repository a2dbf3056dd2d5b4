# A/B: register-cap-aware rows: rotated update R>=5 11 rows (12 warps, 168 cap) vs 12; TTI g pass R 5-6 15 rows (16 warps, 128) vs 16, R 7-8 11 vs 12
out=gpurun_out/r2x_ab.txt; rm -f $out
for rep in 1 2; do for lib in product rows2; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for ks in "rotated 12" "rotated 16" "tti 12" "tti 16"; do set -- $ks
  python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, round(d['value'],1), round(d['roofline']['frac'],3), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
  done; done; done
unset SDMP_LIB
