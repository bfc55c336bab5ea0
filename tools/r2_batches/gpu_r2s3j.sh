#!/bin/bash
set -u
OUT=gpurun_out/r2s3j
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
for v in cur hotf hotn hotu; do lib $v; timeout 600 python tools/time_ops.py c4 c5 > $OUT/ops_$v.txt 2>&1; done
for v in cur u8 u8t4 u16; do lib $v; timeout 300 python tools/time_e2e.py > $OUT/e2e_$v.txt 2>&1; done
echo done > $OUT/DONE
