#!/bin/bash
set -u
OUT=gpurun_out/r2s3g
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 300 python tools/time_e2e.py > $OUT/e2e.txt 2>&1
TCS_E2E_TRACE=1 timeout 300 python tools/time_e2e.py > $OUT/e2e_trace.txt 2>&1
for v in cur nodeep tfd5 tf64 tf64d5; do lib $v; timeout 600 python tools/time_tf32.py > $OUT/tf32_$v.txt 2>&1; done
echo done > $OUT/DONE
