# A/B: 7-row tiles (8 warps, 255-register cap) for the wide velocity / stress /
# TTI-update ops (ab/libsdmp_ty7.so) vs product 8-row tiles (9 warps, 168 cap)
out=gpurun_out/r2q_ab.txt; rm -f $out
for lib in product ty7; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_ty7.so; fi
  for ks in "elastic 12" "elastic 16" "visco 12" "visco 16" "tti 12" "tti 16"; do set -- $ks
    python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, round(d['value'],1), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
  done; done
unset SDMP_LIB
