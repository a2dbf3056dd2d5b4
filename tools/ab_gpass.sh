# A/B: TTI SO-8 g-pass launch shapes (rows per CTA x CTAs per SM): product
# 8 x 2; g4c4 4 x 4; g8c3 8 x 3; g6c3 6 x 3.  Parity of each variant on the
# TTI GPU tests first -> gpurun_out/round2_ab_gpass.txt
out=gpurun_out/round2_ab_gpass.txt; rm -f $out
for lib in g4c4 g8c3 g6c3; do
  SDMP_LIB=ab/libsdmp_$lib.so timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_cabi_gpu.py -q -k "tti" 2>&1 | tail -1 | sed "s/^/$lib tests: /" >> $out
done
for rep in 1 2; do for lib in product g4c4 g8c3 g6c3; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for shp in 512,512,512 768,768,768; do
  timeout 300 python bench.py --kernel tti --so 8 --shape $shp --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'tti SO-8 $shp', round(d['value'],2), round(d['roofline']['frac'],3))" >> $out
  done
done; done
unset SDMP_LIB
cat $out
