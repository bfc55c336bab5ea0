#!/bin/bash
set -u
OUT=gpurun_out/r2s3h
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
timeout 300 python tools/time_encode.py > $OUT/encode.txt 2>&1
timeout 300 python tools/time_e2e.py > $OUT/e2e.txt 2>&1
TCS_E2E_TRACE=1 timeout 300 python tools/time_e2e.py > $OUT/e2e_trace.txt 2>&1
for v in cur nopdl; do lib $v; timeout 300 python tools/time_small.py 3 > $OUT/small_$v.txt 2>&1; done
lib cur; timeout 600 python tools/time_ops.py c3 c4 c5 > $OUT/ops.txt 2>&1
echo done > $OUT/DONE
