# A/B: CTA rasterisation of the streaming kernels (SDMP_SWZ = band width in
# z-tiles; product 0 = plain order).  Oracle check of each variant on grids
# with many z-tiles first, then bench lines at the big planes where the
# y-halo re-reads show (checksums of 6 steps on grids with 17+ z-tiles must
# equal the product's bit for bit) -> gpurun_out/round2_ab_swz.txt
out=gpurun_out/round2_ab_swz.txt; rm -f $out
for lib in product swz2 swz4 swz8; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for k in "acoustic 8 40,48,1100" "elastic 8 40,48,1100" "visco 16 40,40,1100" "tti 8 28,32,1100" "acoustic 16 40,48,1100"; do
    set -- $k
    timeout 600 python -m paper_2312_13094_b200.bench_cli --kernel $1 --so $2 --shape $3 --tn 6 --json 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib checksum $1 SO-$2', repr(d['checksum']))" >> $out 2>&1
  done
done
for rep in 1 2; do for lib in product swz2 swz4 swz8; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for k in "acoustic 8 1024,1024,1024" "acoustic 16 1024,1024,1024" "elastic 8 1024,1024,1024" "elastic 8 512,512,512" "visco 16 512,512,1024" "tti 8 512,512,512"; do
    set -- $k
    timeout 300 python bench.py --kernel $1 --so $2 --shape $3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1 SO-$2 $3', round(d['value'],2), round(d['roofline']['frac'],3))" >> $out
  done
done; done
unset SDMP_LIB
cat $out
