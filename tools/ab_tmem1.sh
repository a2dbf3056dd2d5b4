# A/B: single-load star_tmem1 (u0 crosses HBM once; y/z partial sums parked for R planes)
# at tile heights 16 (partial sums in TMEM) / 20 / 24 (in shared memory) vs star_tmem (product)
out=gpurun_out/r4o_ab.txt; rm -f $out
for rep in 1 2; do for lib in product t1_16 t1_20 t1_24; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for so in 14 16; do
    timeout 120 python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
for so in 4 8 12; do timeout 120 python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('product(reordered)', 'SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out; done
for so in 8 16; do timeout 300 python bench.py --kernel damped --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('product(reordered) damped', 'SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out; done
for lib in t1_16 t1_20 t1_24; do SDMP_LIB=ab/libsdmp_$lib.so /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:star_tmem1 -c 1 --csv python bench.py --kernel acoustic --so 16 --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | grep -v "^{" | tail -3 | cut -d, -f13- >> $out; done
