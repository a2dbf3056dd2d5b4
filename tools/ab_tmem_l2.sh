# A/B: L2 eviction hints on star_tmem's TMA loads (acoustic SO-14/16, 1024^3):
# l2a front evict_last; l2b + centre evict_first; l2c + u2/m evict_first
out=gpurun_out/r4h_ab.txt; rm -f $out
for rep in 1 2; do for lib in product l2a l2b l2c; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  for so in 14 16; do
    timeout 120 python bench.py --kernel acoustic --so $so --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'SO-$so', round(d['value'],1), round(d['roofline']['frac'],3))" >> $out
  done; done; done
unset SDMP_LIB
for lib in l2a l2b; do SDMP_LIB=ab/libsdmp_$lib.so /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:star_tmem -c 1 --csv python bench.py --kernel acoustic --so 16 --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | grep -v "^{" | tail -4 >> $out; done
