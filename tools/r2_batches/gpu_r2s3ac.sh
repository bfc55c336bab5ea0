#!/bin/bash
set -u
OUT=gpurun_out/r2s3ac
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for v in cur c32off c32_8k c32_6k; do lib $v; timeout 300 python tools/time_encode.py c5 > $OUT/encode_$v.txt 2>&1; done
echo done > $OUT/DONE
