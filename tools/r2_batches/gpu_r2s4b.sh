#!/bin/bash
# encode: entries write column_indices (no distinct-column list / copy pass), shift for the block index,
# scatter register budget for 3 CTAs/SM; bitmap 4 entries in flight at 3 CTAs/SM
set -u
OUT=gpurun_out/r2s4b
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 700 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_dropin.py tests/test_gpu_cli.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for v in base cur noce sc1 u8; do lib $v; timeout 150 python tools/time_encode.py > $OUT/encode_$v.txt 2>&1; done
lib cur; timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv python tools/profile_ops.py c3 encode > $OUT/launches_c3.csv 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv python tools/profile_ops.py c5 encode > $OUT/launches_c5.csv 2>&1
echo done > $OUT/DONE
