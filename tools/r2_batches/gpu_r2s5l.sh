#!/bin/bash
# session 5 (experiment, not in the tree): window_sort_rank's column loads batched 4 per thread with the row-order
# predecessor by SHFL (variant sortb, patch in profiles/r2_encode.txt) vs the tree (cur): parity on the variant, encode timing
set -u
OUT=gpurun_out/r2s5l
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib sortb; timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -x -q > $OUT/pytest_sortb.log 2>&1; echo rc=$? >> $OUT/pytest_sortb.log
for r in 1 2; do for v in cur sortb; do lib $v; timeout 200 python tools/time_encode.py > $OUT/encode_${v}_$r.txt 2>&1; done; done
echo done > $OUT/DONE
