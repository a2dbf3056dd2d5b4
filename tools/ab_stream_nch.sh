# usage: bash tools/ab_stream_nch.sh ; stream-engine chunk-picker per-CTA cost sweep (SDMP_STREAM_CTA_PLANES)
for b in 0 4 8 16 0; do export SDMP_STREAM_CTA_PLANES=$b
  for k in "tti 8 512" "elastic 8 512" "visco 16 512" "rotated 8 512" "damped 8 1024"; do set -- $k
  python bench.py --kernel $1 --so $2 --shape $3,$3,$3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('b=$b', '$1', $2, $3, round(d['value'],2), round(d['roofline']['frac'],3))"
  done
done
