# A/B: single-pass kernels unrolled by 2 planes (product) vs 1 (ab/libsdmp_u1.so), and
# the unrolled single pass at SO-6/8 (ab/libsdmp_f4u.so) against the two passes
out=gpurun_out/r2u_ab.txt; rm -f $out
for lib in product u1 f4u; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for ks in "tti 4" "tti 6" "tti 8" "rotated 4" "rotated 6" "rotated 8"; do set -- $ks
    python bench.py --kernel $1 --so $2 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done
unset SDMP_LIB
