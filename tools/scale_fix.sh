source tools/scale_all.sh --defs-only
run 4 acoustic 8 - full ac_n4_full
run 4 acoustic 8 - diagonal ac_n4_diagonal
SDMP_GRAPH=0 run 2 elastic 8 1024,1024,1024 diagonal el_n2_diag_nograph
run 2 elastic 8 1024,1024,1024 diagonal el_n2_diagonal
