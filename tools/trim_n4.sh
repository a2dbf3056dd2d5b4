# Per-field halo radii (stress faces only along their derivative axes): the
# multi-rank bitwise suite on real GPUs, then the elastic / visco lines
# (C4 diagonal + full, C5 full) at N = 2 and 4 -> gpurun_out/round2_trim/
O=gpurun_out/round2_trim; mkdir -p $O
timeout 1500 python -m pytest tests/test_multigpu.py -q --timeout 1400 > $O/pytest_multigpu.txt 2>&1
echo "rc=$?" >> $O/pytest_multigpu.txt
SCALE_OUT=$O ONLY='^(el|visco)_' bash tools/scale_round2.sh
