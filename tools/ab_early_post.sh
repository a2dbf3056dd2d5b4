# Early flag release in full mode (post of a phase depends only on the
# previous phase's OWNED slabs): multi-rank bitwise suite, then a same-box
# A/B (SDMP_EARLY_POST=1 default vs 0) of C5 visco SO-16 and C4 elastic in
# full mode at N = 4 (and N = 2) -> gpurun_out/round2_ab_early_post/
O=gpurun_out/round2_ab_early_post; mkdir -p $O
timeout 1500 python -m pytest tests/test_multigpu.py -q --timeout 1400 > $O/pytest_multigpu.txt 2>&1
echo "rc=$?" >> $O/pytest_multigpu.txt
NG=$(nvidia-smi -L | wc -l)
for rep in 1 2; do
  for ep in 1 0; do
    export SDMP_EARLY_POST=$ep
    for N in 4 2; do
      [ $NG -lt $N ] && continue
      L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2966$N"
      if [ "$N" = 2 ]; then export CUDA_VISIBLE_DEVICES=0,1; else unset CUDA_VISIBLE_DEVICES; fi
      timeout 600 $L bench.py --gpus $N --kernel visco --so 16 --shape 1024,1024,1024 --mode full --steps 20 --warmup 3 --no-cpu-baseline 2>>$O/err.log | tail -1 > $O/visco_n${N}_ep${ep}_$rep.json
      timeout 600 $L bench.py --gpus $N --kernel elastic --so 8 --shape 1024,1024,1024 --mode full --steps 20 --warmup 3 --no-cpu-baseline 2>>$O/err.log | tail -1 > $O/el_n${N}_ep${ep}_$rep.json
    done
  done
done
unset CUDA_VISIBLE_DEVICES
python - $O <<'PY' > $O/summary.txt
import json, glob, os, sys
for f in sorted(glob.glob(sys.argv[1] + "/*.json")):
    try:
        d = json.load(open(f)); h = d["halo"]
        print(os.path.basename(f), round(d["value"], 1), "ms", round(d["ms_per_step"], 3),
              "exposed", round(h["exposed_frac"], 4), "compute-only ms", round(h["compute_only_step_ms"], 3))
    except Exception as e:
        print(os.path.basename(f), "failed", e)
PY
cat $O/summary.txt; tail -2 $O/pytest_multigpu.txt
