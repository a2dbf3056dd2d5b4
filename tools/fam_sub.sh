out=$1; rm -f $out
run() { python bench.py --kernel $1 --so $2 $3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> $out; }
for k in elastic visco tti rotated; do for so in 8 16; do run $k $so "--shape 512,512,512"; done; done
python - $out <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d = json.loads(l); r = d["roofline"]
    acts = [round(a["ms"],3) for a in d["step_actions"] if a["ms"] > 0.05]
    print(d["config"]["workload"], round(d["value"], 1), round(r["frac"], 3), acts)
PY
