#!/bin/bash
set -u
OUT=gpurun_out/r2s3o
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
for v in cur tf5 tf6; do lib $v; timeout 600 python tools/time_tf32.py > $OUT/tf32_$v.txt 2>&1; done
echo done > $OUT/DONE
