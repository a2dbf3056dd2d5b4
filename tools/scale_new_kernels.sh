# Multi-GPU lines for the kernels added late in round 2: acoustic SO-16 (star_tmem, 1024^3 per GPU)
# and the 16-row single-pass rotated operator (SO-8, 1024^3 global), full and diagonal modes
out=gpurun_out/r5h_scale.txt; rm -f $out
for N in 2 4; do
  L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2974$N"
  if [ "$N" = 2 ]; then export CUDA_VISIBLE_DEVICES=0,1; else unset CUDA_VISIBLE_DEVICES; fi
  for m in full diagonal; do for k in "acoustic 16 -" "rotated 8 1024,1024,1024"; do set -- $k
    shp=""; [ "$3" != "-" ] && shp="--shape $3"
    timeout 600 $L bench.py --gpus $N --kernel $1 --so $2 $shp --mode $m --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d.get('halo') or {}; print('N=$N $m', '$1 SO-$2', round(d['value'],1), 'GPts/s frac', round(d['roofline']['frac'],3), 'exposed', round(h.get('exposed_frac',0),4), 'e2e', round(d['e2e']['value'],1))" >> $out
  done; done
done
unset CUDA_VISIBLE_DEVICES
