# A/B on a 4-GPU box: decomposition topology (x/y splits) per family, full mode
out=gpurun_out/r4s_ab.txt; rm -f $out
for N in 2 4; do
  L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2973$N"
  if [ "$N" = 2 ]; then export CUDA_VISIBLE_DEVICES=0,1; T="2,1,1 1,2,1"; else unset CUDA_VISIBLE_DEVICES; T="2,2,1 1,4,1 4,1,1"; fi
  for t in $T; do for k in "visco 16" "elastic 8" "acoustic 8"; do set -- $k
    shp="--shape 1024,1024,1024"; [ $1 = acoustic ] && shp=""
    timeout 600 $L bench.py --gpus $N --kernel $1 --so $2 $shp --topology $t --mode full --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d.get('halo') or {}; print('N=$N topo=$t', '$1', $2, round(d['value'],1), 'exposed', round(h.get('exposed_frac',0),4), 'step', round(d['ms_per_step'],3))" >> $out
  done; done
done
unset CUDA_VISIBLE_DEVICES
