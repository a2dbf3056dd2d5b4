# 4-GPU box: diagonal / basic with the batched SM posts (default) vs copy
# engines, and the 8-rank bench path (2 ranks per GPU, gloo control plane)
O=gpurun_out/round2_scale_b; mkdir -p $O
L="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641"
for eng in batch ce; do
  export SDMP_COPY_ENGINE=$eng
  timeout 600 $L bench.py --gpus 4 --kernel elastic --so 8 --shape 1024,1024,1024 --mode diagonal --steps 20 --warmup 3 --no-cpu-baseline 2>$O/err_el_$eng.log | tail -1 > $O/el_n4_diagonal_$eng.json
  timeout 600 $L bench.py --gpus 4 --mode diagonal --steps 20 --warmup 3 --no-cpu-baseline 2>$O/err_ac_$eng.log | tail -1 > $O/ac_n4_diagonal_$eng.json
  timeout 600 $L bench.py --gpus 4 --mode basic --steps 20 --warmup 3 --no-cpu-baseline 2>$O/err_acb_$eng.log | tail -1 > $O/ac_n4_basic_$eng.json
done
unset SDMP_COPY_ENGINE
timeout 600 $L bench.py --gpus 4 --steps 20 --warmup 3 --no-cpu-baseline 2>$O/err_ac_full.log | tail -1 > $O/ac_n4_full.json
# 8 ranks on 4 GPUs: the (4,2,1) topology of the driver's 8-GPU run, functional check only
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29642 bench.py --gpus 8 --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_8ranks_on_4gpus.json 2> $O/err_8ranks.log
echo "8-rank rc=$?" >> $O/err_8ranks.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29643 bench.py --impl reference --gpus 8 --steps 2 --warmup 1 > $O/ref_8ranks.json 2> $O/err_ref8.log
python tools/scale_summary.py $O > $O/summary.txt 2>&1
