# bitwise multi-GPU == single-GPU at (near) BASELINE sizes; N = $1
N=$1
L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N"
mkdir -p gpurun_out/fullsize
for m in full diagonal basic; do $L tools/fullsize_multigpu.py --mode $m 2>>gpurun_out/fullsize/err.log | tail -1 | tee -a gpurun_out/fullsize/n$N.jsonl | cut -c1-120; done
$L tools/fullsize_multigpu.py --kernel elastic --shape 1024,1024,1024 --mode diagonal 2>>gpurun_out/fullsize/err.log | tail -1 | tee -a gpurun_out/fullsize/n$N.jsonl | cut -c1-120
$L tools/fullsize_multigpu.py --kernel tti --shape 1024,1024,1024 --mode full 2>>gpurun_out/fullsize/err.log | tail -1 | tee -a gpurun_out/fullsize/n$N.jsonl | cut -c1-120
$L tools/fullsize_multigpu.py --kernel visco --shape 768,768,768 --mode full 2>>gpurun_out/fullsize/err.log | tail -1 | tee -a gpurun_out/fullsize/n$N.jsonl | cut -c1-120
grep -c '"all_equal": true, "traces_equal": true' gpurun_out/fullsize/n$N.jsonl
