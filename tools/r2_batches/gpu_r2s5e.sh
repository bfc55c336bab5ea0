#!/bin/bash
# session 5: source-level ncu of the C5 AGNN attention, the C3 SDDMM and the C1/C2 burst kernels
set -u
KEEP_REP=1 bash tools/gpu_profiles.sh r2s5e c5:attend:fp16:32 c3:sddmm:fp16:32 c1:spmm:fp16:128 c1:sddmm:fp16:32
echo done > gpurun_out/r2s5e/DONE
