# usage: bash tools/scale_families.sh N ; BASELINE C3/C4/C5 configs on N GPUs
N=$1
run() {  # kernel so shape mode
  if [ "$N" = 1 ]; then L="python"; else L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"; fi
  timeout 900 $L bench.py --gpus $N --kernel $1 --so $2 --shape $3 --mode $4 --steps 10 --warmup 3 --no-cpu-baseline 2>gpurun_out/err_$1_$N_$4.log | tail -1 > gpurun_out/fam_$1_n${N}_$4.json
  python -c "
import json; d=json.load(open('gpurun_out/fam_$1_n${N}_$4.json')); h=d.get('halo') or {}
print('$1 N=$N $4', round(d['value'],2), 'ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), 'halo', {k: h[k] for k in list(h)[:6]})" || tail -5 gpurun_out/err_$1_$N_$4.log
}
mkdir -p gpurun_out
if [ "$N" != 1 ]; then run tti 8 1536,1536,1536 full; fi
run elastic 8 1024,1024,1024 diagonal
if [ "$N" != 1 ]; then run visco 16 1024,1024,1024 full; fi
