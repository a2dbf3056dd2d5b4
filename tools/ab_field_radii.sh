# A/B on one 4-GPU box: per-field halo radii (default) vs every field on every
# face (SDMP_FIELD_RADII=0), C4 elastic diagonal and C5 visco full at N = 4,
# alternating, two rounds -> gpurun_out/round2_ab_field_radii/
O=gpurun_out/round2_ab_field_radii; mkdir -p $O
L="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651"
for rep in 1 2; do
  for fr in 1 0; do
    export SDMP_FIELD_RADII=$fr
    timeout 600 $L bench.py --gpus 4 --kernel elastic --so 8 --shape 1024,1024,1024 --mode diagonal --steps 20 --warmup 3 --no-cpu-baseline 2>>$O/err.log | tail -1 > $O/el_diag_fr${fr}_$rep.json
    timeout 600 $L bench.py --gpus 4 --kernel visco --so 16 --shape 1024,1024,1024 --mode full --steps 20 --warmup 3 --no-cpu-baseline 2>>$O/err.log | tail -1 > $O/visco_full_fr${fr}_$rep.json
  done
done
python - $O <<'PY' > $O/summary.txt
import json, glob, os, sys
for f in sorted(glob.glob(sys.argv[1] + "/*.json")):
    try:
        d = json.load(open(f)); h = d["halo"]
        print(os.path.basename(f), round(d["value"], 1), "ms", round(d["ms_per_step"], 3),
              "exposed", round(h["exposed_frac"], 4), "compute-only ms", round(h["compute_only_step_ms"], 3),
              "sent MB", round(h["halo_bytes_sent_per_step_rank0"] / 1e6, 1))
    except Exception as e:
        print(os.path.basename(f), "failed", e)
PY
cat $O/summary.txt
