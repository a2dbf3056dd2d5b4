# A/B: elastic stress tile rows at R <= 4 (product 8; st12, st16), at 512^3
# and 1024^3 (where the stress kernel re-reads y halos: 1.21x algorithmic).
# Variant parity on the elastic GPU tests first -> gpurun_out/round2_ab_stress_rows.txt
out=gpurun_out/round2_ab_stress_rows.txt; rm -f $out
for lib in st12 st16; do
  SDMP_LIB=ab/libsdmp_$lib.so timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_cabi_gpu.py -q -k "elastic or visco" 2>&1 | tail -1 | sed "s/^/$lib tests: /" >> $out
done
for rep in 1 2; do for lib in product st12 st16; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for shp in 512,512,512 1024,1024,1024; do
  timeout 300 python bench.py --kernel elastic --so 8 --shape $shp --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'elastic SO-8 $shp', round(d['value'],2), round(d['roofline']['frac'],3))" >> $out
  done
done; done
unset SDMP_LIB
cat $out
