source tools/gpu/abl_tcc2.sh
export ABL_ARGS=--all
run cp4 -DENSI_TCC_CPAIRS_MAX=4
run cp2 -DENSI_TCC_CPAIRS_MAX=2
run cp3 -DENSI_TCC_CPAIRS_MAX=3
