#!/bin/bash
set -u
OUT=gpurun_out/r2s3m
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
for v in cur pf32 pf128; do lib $v; timeout 600 python tools/time_tf32.py > $OUT/tf32_$v.txt 2>&1; done
for v in cur pfh64 pfh128 hotf2 hotn2; do lib $v; timeout 600 python tools/time_ops.py c3 c4 c5 > $OUT/ops_$v.txt 2>&1; done
echo done > $OUT/DONE
