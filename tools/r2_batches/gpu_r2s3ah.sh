#!/bin/bash
set -u
OUT=gpurun_out/r2s3ah
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2 3; do for v in base_e2e cur; do lib $v; timeout 300 python tools/time_e2e.py >> $OUT/e2e_$v.txt 2>&1; done; done
lib cur; TCS_E2E_TRACE=1 timeout 300 python tools/time_e2e.py > $OUT/trace_cur.txt 2>&1
timeout 300 python tools/time_encode.py > $OUT/encode.txt 2>&1
echo done > $OUT/DONE
