# A/B on a 4-GPU box: full-mode OWNED x-slabs on the generic kernels (SDMP_THIN_X = 8 / 16) vs streaming kernels (0)
out=gpurun_out/r4r_ab.txt; rm -f $out
for N in 4 2; do
  L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2972$N"
  if [ "$N" = 2 ]; then export CUDA_VISIBLE_DEVICES=0,1; else unset CUDA_VISIBLE_DEVICES; fi
  for t in 0 8 16; do for k in "visco 16" "elastic 8" "acoustic 8" "tti 8"; do set -- $k
    shp="--shape 1024,1024,1024"; [ $1 = acoustic ] && shp=""; [ $1 = tti ] && shp="--shape 1536,1536,1536"
    [ $1 = tti ] && [ $N = 2 ] && continue
    SDMP_THIN_X=$t timeout 600 $L bench.py --gpus $N --kernel $1 --so $2 $shp --mode full --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d.get('halo') or {}; print('N=$N thin_x=$t', '$1', $2, round(d['value'],1), 'exposed', round(h.get('exposed_frac',0),4), 'step', round(d['ms_per_step'],3))" >> $out
  done; done
done
unset CUDA_VISIBLE_DEVICES
