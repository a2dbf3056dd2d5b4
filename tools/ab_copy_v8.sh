# A/B on 2 GPUs: batched post kernel with 32-byte (product) vs 16-byte (ab/libsdmp_v4.so) stores
out=gpurun_out/r3g_ab.txt; rm -f $out
for lib in product v4; do
  if [ $lib = product ]; then unset SDMP_LIB; else export SDMP_LIB=ab/libsdmp_$lib.so; fi
  python tools/nvlink_bw.py 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l)
    if 'batched' in d['engine'] or 'contiguous' in d['case']: print('$lib', d['case'], d.get('whole_z'), round(d['gbs'],1))" >> $out
  for rep in 1 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 2 --kernel elastic --so 8 --shape 1024,1024,1024 --mode diagonal --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d['halo']
print('$lib elastic diag N=2', round(d['value'],1), 'exposed', round(100*h['exposed_frac'],2), '%', 'link', round(h['link_gbs_rank0'] or 0))" >> $out
  done
done
unset SDMP_LIB
timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "four_ranks_xy or listing4" > gpurun_out/r3g_multi.log 2>&1; echo rc=$? >> gpurun_out/r3g_multi.log
