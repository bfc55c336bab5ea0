#!/bin/bash
# Session batch: GPU suite, small-config timings (+ launch floor), e2e
# pipeline timing and trace, ncu captures of the small-config kernels.
set -u
OUT=gpurun_out/r2s3c
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
timeout 300 python tools/time_small.py 3 > $OUT/small.txt 2>&1
timeout 300 python tools/time_e2e.py > $OUT/e2e.txt 2>&1
TCS_E2E_TRACE=1 timeout 300 python tools/time_e2e.py > $OUT/e2e_trace.txt 2>&1
KEEP_REP=0 bash tools/gpu_profiles.sh r2s3c/ncu c1:spmm:fp16:128 c1:sddmm:fp16:32 c1:spmm:tf32:128 c1:sddmm:tf32:32
echo done > $OUT/DONE
