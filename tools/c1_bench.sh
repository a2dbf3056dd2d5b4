# C1 (acoustic SO-8 256^3, 200 steps) bench lines in diagonal and full mode
for m in diagonal full; do python bench.py --shape 256,256,256 --mode $m --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1; done
