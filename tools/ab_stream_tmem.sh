# A/B: stream-engine x-window in tensor memory (ab/libsdmp_tm*.so) vs registers (product)
out=gpurun_out/r4b_ab.txt; rm -f $out
for lib in product tm5 tm5w; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for k in "tti 12 512" "tti 16 512" "rotated 12 512" "rotated 16 512" "elastic 12 512" "elastic 16 512" "visco 12 512" "visco 16 512" "damped 16 1024"; do set -- $k
    timeout 300 python bench.py --kernel $1 --so $2 --shape $3,$3,$3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1', $2, round(d['value'],2), round(d['roofline']['frac'],3))" >> $out
  done
done
unset SDMP_LIB
