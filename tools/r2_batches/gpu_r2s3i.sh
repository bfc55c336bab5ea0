#!/bin/bash
set -u
OUT=gpurun_out/r2s3i
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
for v in cur nohot; do lib $v; timeout 600 python tools/time_ops.py c3 c4 c5 > $OUT/ops_$v.txt 2>&1; done
for v in cur nohot; do lib $v; AB_LAYERS=1 timeout 600 python tools/bench_layers.py > $OUT/layers_$v.txt 2>&1; done
for v in cur st3; do lib $v; timeout 300 python tools/time_e2e.py > $OUT/e2e_$v.txt 2>&1; done
lib cur; TCS_E2E_TRACE=1 timeout 300 python tools/time_e2e.py > $OUT/e2e_trace.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
echo done > $OUT/DONE
