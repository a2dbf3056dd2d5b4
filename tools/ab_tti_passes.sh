# A/B: TTI SO-8 two-pass variants (front L2 hint on the g / update pass, g-pass tile rows / CTAs, stages)
out=gpurun_out/r5d_ab.txt; rm -f $out
for rep in 1 2; do for lib in product gl2 ul2 g16 g1c gst6; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  timeout 300 python bench.py --kernel tti --so 8 --shape 512,512,512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'tti SO-8', round(d['value'],2), round(d['roofline']['frac'],3))" >> $out
  done; done
unset SDMP_LIB
for lib in product gl2; do if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:stream_kernel -c 2 --csv python bench.py --kernel tti --so 8 --shape 512,512,512 --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | grep -v "^{" | tail -6 | awk -F'","' '{print "'$lib'", $5, $(NF-2), $NF}' >> $out; done
