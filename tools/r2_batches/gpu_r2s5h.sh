#!/bin/bash
# session 5: compute-sanitizer on the final tree (tools/sanitize.sh) plus memcheck of the TF32 tests
# (the deferred-conversion kernels) and racecheck of the AGNN attention
# NOTE: compute-sanitizer is closed on this GPU pool (runs under it returned rc=86 with a refusal message); kept as the command record only.
set -u
bash tools/sanitize.sh r2s5san
OUT=gpurun_out/r2s5san
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tf32 or TF32" > $OUT/memcheck_tf32.log 2>&1; echo "rc=$?" >> $OUT/memcheck_tf32.log
echo done > $OUT/DONE
