#!/bin/bash
# Round-end measurement pass on one GPU box: tools/gpu_round.sh (GPU tests,
# smoke, the bench line, the reference arm, the ncu launch list, ncu --set
# full of the headline SpMM and SDDMM) followed by per-config ncu captures
# (tools/gpu_profiles.sh) whose raw CSVs feed profiles/traffic.json.
#   gpurun --timeout 3600 -- 'bash tools/gpu_final.sh TAG'
set -u
TAG=${1:-final}
bash tools/gpu_round.sh $TAG
KEEP_REP=0 bash tools/gpu_profiles.sh $TAG/ncu c1:spmm:fp16:128 c1:spmm:tf32:128 c1:sddmm:fp16:32 c1:sddmm:tf32:32 \
    c3:spmm:fp16:128 c3:spmm:tf32:128 c3:sddmm:fp16:32 c4:spmm:fp16:128 c5:spmm:fp16:32 c5:sddmm_static:fp16:32
echo done > gpurun_out/$TAG/FINAL_DONE
