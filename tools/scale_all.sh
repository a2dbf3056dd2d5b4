# r02 scaling sweep on a 4-GPU box: acoustic C2 weak (N = 2, 4; basic/diagonal/full)
# and the C3/C4/C5 family configs at N = 2 (GPUs 0,1) and 4.
mkdir -p gpurun_out/scale
run() {  # N kernel so shape mode tag
  N=$1; shift
  if [ "$N" = 1 ]; then L="python"; else L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N"; fi
  if [ "$N" = 2 ]; then export CUDA_VISIBLE_DEVICES=0,1; else unset CUDA_VISIBLE_DEVICES; fi
  shp=""; [ "$3" != "-" ] && shp="--shape $3"
  timeout 900 $L bench.py --gpus $N --kernel $1 --so $2 $shp --mode $4 --steps 20 --warmup 3 --no-cpu-baseline 2>gpurun_out/scale/err_$5.log | tail -1 > gpurun_out/scale/$5.json
  python -c "
import json; d=json.load(open('gpurun_out/scale/$5.json')); h=d.get('halo') or {}
print('$5', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), 'exposed', round(h.get('exposed_frac',0),3), 'link', round(h.get('link_gbs_rank0') or 0))" || tail -3 gpurun_out/scale/err_$5.log
}
[ "$1" = "--defs-only" ] && return 0
for m in basic diagonal full; do run 2 acoustic 8 - $m ac_n2_$m; run 4 acoustic 8 - $m ac_n4_$m; done
run 2 tti 8 1536,1536,1536 full tti_n2_full
run 4 tti 8 1536,1536,1536 full tti_n4_full
run 2 visco 16 1024,1024,1024 full visco_n2_full
run 4 visco 16 1024,1024,1024 full visco_n4_full
run 2 elastic 8 1024,1024,1024 diagonal el_n2_diagonal
run 4 elastic 8 1024,1024,1024 diagonal el_n4_diagonal
run 4 elastic 8 1024,1024,1024 full el_n4_full
