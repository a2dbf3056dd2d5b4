# TTI / rotated GPts/s vs grid size on one GPU: at 96^3-128^3 every array of
# both passes fits in the 126 MB L2, so the rate there is the non-HBM
# (shared-memory / issue) ceiling of the two-pass kernels (r04 analysis).
out=${1:-gpurun_out/tti_floor.jsonl}; rm -f $out
for k in tti rotated; do for n in 512 384 256 160 128 96; do
python bench.py --kernel $k --so 8 --shape $n,$n,$n --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> $out
done; done
python - "$out" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l); r = d["roofline"]
    print(d["config"]["workload"], round(d["value"], 1), "GPts/s", round(r["frac"], 3),
          "launch_ms", round(r["launch_ms"], 4))
PY
