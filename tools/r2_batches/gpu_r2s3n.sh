#!/bin/bash
set -u
OUT=gpurun_out/r2s3n
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
for v in cur nopf; do lib $v; timeout 600 python tools/time_tf32.py > $OUT/tf32_$v.txt 2>&1; done
for v in cur nopf hotf2 hotn2; do lib $v; timeout 600 python tools/time_ops.py c3 c4 c5 > $OUT/ops_$v.txt 2>&1; done
lib cur; timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
echo done > $OUT/DONE
