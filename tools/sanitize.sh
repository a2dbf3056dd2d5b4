# compute-sanitizer over smoke(), every family x mode (single process, small
# grids) and a 2-rank oversubscribed full-mode run (CUDA IPC peer stores,
# release/acquire flags, 3-stream joins).  Logs -> gpurun_out/san_*.log
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out
export SDMP_TIMEOUT_MS=600000 SDMP_GRAPH=1
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 7 --log-file $O/san_${tool}_smoke.log \
    python -c "import __graft_entry__ as g; g.smoke()" > $O/san_${tool}_smoke.out 2>&1
  echo "smoke $tool rc=$?" >> $O/san_summary.txt
done
for tool in memcheck racecheck synccheck; do
  FAMILIES=acoustic,damped,rotated,tti,elastic,elastic_col,visco STEPS=2 timeout 2400 \
    $CS --tool $tool --error-exitcode 7 --log-file $O/san_${tool}_families.log \
    python tools/sanitize_families.py > $O/san_${tool}_families.out 2>&1
  echo "families $tool rc=$?" >> $O/san_summary.txt
done
for tool in memcheck synccheck; do
  FAMILIES=acoustic,tti,elastic TOPO=2,1,1 SHAPE=40,20,24 STEPS=3 SDMP_DIST_BACKEND=gloo \
    timeout 2400 $CS --tool $tool --target-processes all --error-exitcode 7 \
    --log-file $O/san_${tool}_2rank_%p.log \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
    --master-port=29601 tests/mp_worker.py > $O/san_${tool}_2rank.out 2>&1
  echo "2-rank $tool rc=$?" >> $O/san_summary.txt
done
