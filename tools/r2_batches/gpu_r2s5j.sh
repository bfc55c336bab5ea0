#!/bin/bash
# session 5: source-level ncu of the C5 encode (window_sort_big / warp / small, scatter)
set -u
KEEP_REP=1 bash tools/gpu_profiles.sh r2s5j c5:encode:fp16:0
echo done > gpurun_out/r2s5j/DONE
