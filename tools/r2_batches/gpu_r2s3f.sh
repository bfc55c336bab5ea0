#!/bin/bash
set -u
OUT=gpurun_out/r2s3f
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
timeout 300 python tools/time_encode.py > $OUT/encode.txt 2>&1
timeout 300 python tools/time_e2e.py > $OUT/e2e.txt 2>&1
TCS_E2E_TRACE=1 timeout 300 python tools/time_e2e.py > $OUT/e2e_trace.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $OUT/e2e_launches.csv python tools/profile_e2e.py > $OUT/ncu_e2e.log 2>&1
echo done > $OUT/DONE
