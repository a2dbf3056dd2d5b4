# Multi-GPU lines on whatever box this runs on (N = 2 and, with >= 4 GPUs,
# N = 4): acoustic C2 weak scaling in all three modes, C3 TTI 1536^3 full,
# C4 elastic 1024^3 diagonal (+ full), C5 visco SO-16 1024^3 full.  Each line
# carries the halo block (exposed time, bytes, link rate, NVML NVLink
# counters).  -> gpurun_out/round2_scale/*.json + summary.txt
O=${SCALE_OUT:-gpurun_out/round2_scale}; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
run() {  # N kernel so shape mode tag   (ONLY=<regex>: run matching tags only)
  N=$1; shift
  if [ -n "$ONLY" ] && ! echo "$5" | grep -Eq "$ONLY"; then return; fi
  L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N"
  if [ "$N" = 2 ]; then export CUDA_VISIBLE_DEVICES=0,1; else unset CUDA_VISIBLE_DEVICES; fi
  shp=""; [ "$3" != "-" ] && shp="--shape $3"
  timeout 900 $L bench.py --gpus $N --kernel $1 --so $2 $shp --mode $4 --steps 20 --warmup 3 --no-cpu-baseline 2>$O/err_$5.log | tail -1 > $O/$5.json
  python - "$O/$5.json" "$5" >> $O/summary.txt <<'PY' || tail -3 $O/err_$5.log >> $O/summary.txt
import json, sys
d = json.load(open(sys.argv[1])); h = d.get("halo") or {}; nv = h.get("nvlink_counters_rank0")
nv = nv if isinstance(nv, dict) else {}
print(sys.argv[2], round(d["value"], 1), "GPts/s ms", round(d["ms_per_step"], 3), "frac",
      round(d["roofline"]["frac"], 3), "e2e", round(d["e2e"]["value"], 1), "exposed",
      round(h.get("exposed_frac", 0), 4), "sent MB", round(h.get("halo_bytes_sent_per_step_rank0", 0) / 1e6, 1),
      "link GB/s", round(h.get("link_gbs_rank0") or 0), "nvml tx MB/step",
      round((nv.get("tx_bytes_per_step") or 0) / 1e6, 1), "nvml GB/s in window",
      round(nv.get("tx_gbs_during_transfer") or 0))
PY
}
for N in 2 4; do
  [ $NG -lt $N ] && continue
  for m in basic diagonal full; do run $N acoustic 8 - $m ac_n${N}_$m; done
  run $N tti 8 1536,1536,1536 full tti_n${N}_full
  run $N elastic 8 1024,1024,1024 diagonal el_n${N}_diagonal
  run $N elastic 8 1024,1024,1024 full el_n${N}_full
  run $N visco 16 1024,1024,1024 full visco_n${N}_full
done
cat $O/summary.txt
