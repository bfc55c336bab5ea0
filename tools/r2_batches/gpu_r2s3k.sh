#!/bin/bash
set -u
OUT=gpurun_out/r2s3k
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
for v in cur b256 s256 bs256; do lib $v; timeout 300 python tools/time_encode.py > $OUT/encode_$v.txt 2>&1; done
for v in cur bs256; do lib $v; timeout 300 python tools/time_e2e.py > $OUT/e2e_$v.txt 2>&1; done
lib cur
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $OUT/e2e_launches.csv python tools/profile_e2e.py > $OUT/ncu_e2e.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $OUT/enc_c3_launches.csv python tools/profile_ops.py c3 encode > $OUT/ncu_enc.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
echo done > $OUT/DONE
