# A/B on N GPUs: diagonal / basic halo posts by copy engines (ce, product
# default), per-box SM kernels (sm) or one batched SM kernel per post (batch)
N=${1:-2}; out=gpurun_out/r2r_ab_copy_n$N.txt; rm -f $out
L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29633"
for rep in 1 2; do for eng in ce batch sm; do
  export SDMP_COPY_ENGINE=$eng
  for ks in "acoustic 8 - diagonal" "elastic 8 1024,1024,1024 diagonal" "acoustic 8 - basic"; do set -- $ks
    shp=""; [ "$3" != "-" ] && shp="--shape $3"
    timeout 600 $L bench.py --gpus $N --kernel $1 --so $2 $shp --mode $4 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d['halo']
print('$eng', '$1', '$4', round(d['value'],1), 'exposed', round(100*h['exposed_frac'],2), '%', 'post ms', round(h['post_ms_rank0'],3), 'link', round(h['link_gbs_rank0'] or 0))" >> $out
  done; done; done
unset SDMP_COPY_ENGINE
