#!/bin/bash
set -u
OUT=gpurun_out/r2s3d
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
for v in cur bw8 bw16; do lib $v; timeout 300 python tools/time_small.py 3 > $OUT/small_$v.txt 2>&1; done
for v in cur st2 st4; do lib $v; timeout 300 python tools/time_e2e.py > $OUT/e2e_$v.txt 2>&1; done
lib st4; TCS_E2E_TRACE=1 timeout 300 python tools/time_e2e.py > $OUT/e2e_trace_st4.txt 2>&1
for v in cur lo32 ef; do lib $v; timeout 600 python tools/time_ops.py c3 > $OUT/ops_$v.txt 2>&1; done
unset TCS_LIB_PATH
timeout 600 python -m pytest tests/test_gpu_scale.py -q -x -k "pipelined or midsize" > $OUT/pytest_scale.txt 2>&1
echo done > $OUT/DONE
