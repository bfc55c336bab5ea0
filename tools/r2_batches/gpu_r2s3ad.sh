#!/bin/bash
set -u
OUT=gpurun_out/r2s3ad
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_fullsize.py -m gpu -x -q -k "hub or c5 or C5 or config5 or midsize" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for v in cur split0 split4k split8k; do lib $v; timeout 300 python tools/time_encode.py c5 > $OUT/encode_$v.txt 2>&1; done
echo done > $OUT/DONE
