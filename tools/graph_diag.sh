source tools/scale_all.sh --defs-only
run 2 acoustic 8 - diagonal ac_n2_diag_graph
run 2 elastic 8 1024,1024,1024 diagonal el_n2_diag_graph
run 2 acoustic 8 - full ac_n2_full
