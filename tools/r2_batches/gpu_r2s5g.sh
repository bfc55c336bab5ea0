#!/bin/bash
# session 5: claim-ahead persistent loops (variant "ahead": TCS_CLAIM_AHEAD_MAIN/DEEP/ATTEND=1) vs cur:
# parity + layer tests on the variant, then C3/C4/C5 per-op timing and the C5 attention, interleaved
set -u
OUT=gpurun_out/r2s5g
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib ahead; timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_layers.py tests/test_gpu_fullsize.py -m gpu -x -q > $OUT/pytest_ahead.log 2>&1; echo rc=$? >> $OUT/pytest_ahead.log
for r in 1 2; do for v in cur ahead; do lib $v; timeout 400 python tools/time_ops.py c3 c4 c5 > $OUT/ops_${v}_$r.txt 2>&1; timeout 200 python tools/time_attend.py > $OUT/attend_${v}_$r.txt 2>&1; done; done
echo done > $OUT/DONE
