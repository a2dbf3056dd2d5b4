L="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512"
for e in ce; do
SDMP_COPY_ENGINE=$e $L bench.py --gpus 2 --kernel elastic --so 8 --shape 1024,1024,1024 --mode diagonal --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d['halo']; print('$e', d['rank_actions'], round(d['value'],2), round(h['exposed_frac'],3), round(h['post_ms_rank0'],3), h['halo_bytes_sent_per_step_rank0'], [(a['kind'], round(a['ms'],3)) for a in d['step_actions'] if a['kind'] in (10,11,3,4)])"
done
