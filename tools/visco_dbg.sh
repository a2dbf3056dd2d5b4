L="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541"
for args in "--kernel visco --shape 768,768,768 --mode full" "--kernel elastic --shape 1024,1024,1024 --mode full" "--kernel acoustic --mode full"; do
echo "== $args"
$L tools/fullsize_multigpu.py $args 2>>gpurun_out/vdbg_err.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['kernel'], d['shape'], d['mode'], d['all_equal'], d['traces_equal'], [[a==b for a,b in zip(r['hash'], r['hash_single'])] for r in d['ranks']])"
done
source tools/scale_all.sh --defs-only
run 2 acoustic 8 - full ac_n2_full
run 2 visco 16 1024,1024,1024 full visco_n2_full
