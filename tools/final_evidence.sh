# HEAD evidence on one B200 -> gpurun_out/round2_final/ (copied to profiles/ by hand)
O=gpurun_out/round2_final; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?" >> $O/bench_n1.err
python bench.py --impl reference > $O/bench_reference_n1.json 2> $O/bench_reference_n1.err
$NCU --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:sdmp -c 400 --csv \
  --log-file $O/bench_n1_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:star_tma -s 3 -c 1 \
  -o $O/star_tma_so8_1024 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
$NCU -i $O/star_tma_so8_1024.ncu-rep --page raw --csv > $O/star_tma_so8_1024_raw.csv 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
bash tools/family_table.sh > $O/family.txt 2>&1; cp gpurun_out/family_table.jsonl $O/family_table.jsonl
