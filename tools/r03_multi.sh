# r03 multi-GPU refresh on a 4-GPU box: bitwise full-size parity (N = 4) and
# the 4-GPU lines of the families whose kernels changed (x-window unroll)
set +e
bash tools/fullsize_all.sh 4
source tools/scale_all.sh --defs-only
run 4 acoustic 8 - full ac_n4_full
run 4 acoustic 16 - full ac16_n4_full
run 4 tti 8 1536,1536,1536 full tti_n4_full
run 4 visco 16 1024,1024,1024 full visco_n4_full
run 4 elastic 8 1024,1024,1024 full el_n4_full
