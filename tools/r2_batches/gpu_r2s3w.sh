#!/bin/bash
set -u
OUT=gpurun_out/r2s3w
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
for v in cur nopf64; do lib $v; timeout 600 python tools/time_ops.py c3 > $OUT/ops_$v.txt 2>&1; done
lib cur
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $OUT/enc_c5_launches.csv --profile-from-start off python tools/profile_ops.py c5 encode > $OUT/ncu_enc5.log 2>&1
echo done > $OUT/DONE
