L="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29601"
for v in "$@"; do
SDMP_LIB=abtest/libsdmp_$v.so $L bench.py --gpus 4 --kernel elastic --so 8 --shape 1024,1024,1024 --mode diagonal --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d['halo']; print('$v el diag', round(d['value'],1), round(h['exposed_frac'],3), round(h['post_ms_rank0'],3))"
SDMP_LIB=abtest/libsdmp_$v.so $L bench.py --gpus 4 --mode diagonal --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d['halo']; print('$v ac diag', round(d['value'],1), round(h['exposed_frac'],3), round(h['post_ms_rank0'],3))"
done
