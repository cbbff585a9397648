source tools/gpu/abl_tcc2.sh
B="-DENSI_TCC_GROUPS=1 -DENSI_TCC_STAGES=6 -DENSI_TCC_NOCHUNK -DENSI_TCC_LDX8"
run rot $B
run rot_notma $B -DENSI_ABL_NOTMASTORE
cd /tmp/abl_rot && timeout 600 python -m pytest tests/test_gpu_compact.py -x -q -p no:cacheprovider 2>&1 | tail -2
