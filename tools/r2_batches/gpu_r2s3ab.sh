#!/bin/bash
set -u
OUT=gpurun_out/r2s3ab
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_fullsize.py -m gpu -x -q -k "hub or config5 or c5 or C5 or midsize or pipelined" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for v in cur nohub; do lib $v; timeout 300 python tools/time_encode.py > $OUT/encode_$v.txt 2>&1; done
lib cur
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $OUT/enc_c5_launches.csv --profile-from-start off python tools/profile_ops.py c5 encode > $OUT/ncu_enc5.log 2>&1
echo done > $OUT/DONE
