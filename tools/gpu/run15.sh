source tools/gpu/abl_tcc2.sh
B="-DENSI_TCC_GROUPS=1 -DENSI_TCC_STAGES=6 -DENSI_TCC_NOCHUNK -DENSI_TCC_LDX8"
run stsv2 $B -DENSI_TCC_STSV2
run stshalf $B -DENSI_ABL_STSHALF
run base2 $B
cd /tmp/abl_stsv2 && timeout 600 python -m pytest tests/test_gpu_compact.py -x -q -p no:cacheprovider 2>&1 | tail -2
