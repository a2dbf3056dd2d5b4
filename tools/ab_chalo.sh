# A/B: per-tile centre halos (product) vs both halos on every tile (ab/libsdmp_nochalo.so)
out=gpurun_out/r2i_ab.txt; rm -f $out
for rep in 1 2; do for lib in product nochalo; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_nochalo.so; fi
  for ks in "rotated 8" "rotated 16" "tti 8" "tti 16" "elastic 16" "visco 16"; do set -- $ks
    python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, round(d['value'],1), [round(a['ms'],3) for a in d['step_actions'] if a['ms']>0.05])" >> $out
  done; done; done
unset SDMP_LIB
