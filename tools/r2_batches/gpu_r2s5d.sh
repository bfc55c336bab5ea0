#!/bin/bash
# session 5: full GPU suite on the TF32 deferred-conversion build; source-level ncu of the FP16 SpMM kernels (C3 N=128, C5 N=32)
set -u
OUT=gpurun_out/r2s5d
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
KEEP_REP=1 bash tools/gpu_profiles.sh r2s5d c3:spmm:fp16:128 c5:spmm:fp16:32
echo done > $OUT/DONE
