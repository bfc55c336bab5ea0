#!/bin/bash
# window_bitmap: rank pass writes the distinct columns (no bit-scan emit), off-path row-boundary check,
# first batch's columns kept in registers; register budget for 2 vs 3 CTAs/SM; entries in flight 4/6/8
set -u
OUT=gpurun_out/r2s4a
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 700 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for v in base cur m2 m2nk u4m3 u6m3; do lib $v; timeout 150 python tools/time_encode.py > $OUT/encode_$v.txt 2>&1; done
echo done > $OUT/DONE
