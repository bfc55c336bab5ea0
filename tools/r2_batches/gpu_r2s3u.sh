#!/bin/bash
set -u
OUT=gpurun_out/r2s3u
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
for r in 1 2; do for v in cur u6t5 u8t4 u4t6; do lib $v; timeout 300 python tools/time_e2e.py >> $OUT/e2e_$v.txt 2>&1; done; done
echo done > $OUT/DONE
