#!/bin/bash
set -u
OUT=gpurun_out/r2s3q
mkdir -p $OUT
timeout 300 python tools/time_encode.py > $OUT/encode.txt 2>&1
timeout 300 python tools/time_e2e.py > $OUT/e2e.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/enc_c3_launches.csv --profile-from-start off python tools/profile_ops.py c3 encode > $OUT/ncu_enc.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
echo done > $OUT/DONE
