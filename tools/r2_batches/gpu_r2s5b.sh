#!/bin/bash
# session 5: source-level ncu of the TF32 C3 N=128 SpMM and the C3 encode kernels (reports kept for --page source)
set -u
KEEP_REP=1 bash tools/gpu_profiles.sh r2s5b c3:spmm:tf32:128 c3:encode:fp16:0
echo done > gpurun_out/r2s5b/DONE
