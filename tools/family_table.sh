# every family x space order on one B200 -> gpurun_out/family_table.jsonl
out=gpurun_out/family_table.jsonl; rm -f $out
run() { python bench.py --kernel $1 --so $2 $3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> $out; }
for so in 4 8 12 16; do run acoustic $so ""; done
for so in 4 8 16; do run damped $so ""; done
for so in 4 8 16; do run rotated $so "--shape 512,512,512"; done
for so in 8; do run elastic_col $so "--shape 512,512,512"; done
for k in tti elastic visco; do for so in 4 8 12 16; do run $k $so "--shape 512,512,512"; done; done
python - <<'PY'
import json
for l in open("gpurun_out/family_table.jsonl"):
    d = json.loads(l); r = d["roofline"]
    print(d["config"]["workload"], round(d["value"], 1), round(r["frac"], 3), r["bytes_per_point"])
PY
