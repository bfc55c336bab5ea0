#!/bin/bash
# session 5: the global-memory hub bitmap's popcount / prefix passes as coalesced warp scans (cur) vs thread-contiguous
# runs (gbm0): encode parity (golden, hub windows of wide column spaces, C5 full size), then C3/C5 encode timing interleaved
set -u
OUT=gpurun_out/r2s5k
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_cli.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2; do for v in gbm0 cur; do lib $v; timeout 200 python tools/time_encode.py > $OUT/encode_${v}_$r.txt 2>&1; done; done
echo done > $OUT/DONE
