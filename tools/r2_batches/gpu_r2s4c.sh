#!/bin/bash
# encode: scatter claims its next unit while writing the current one (noclaim = A/B); sort-rank kernels
# no longer write the distinct-column list; e2e on the new encode
set -u
OUT=gpurun_out/r2s4c
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 700 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_dropin.py tests/test_gpu_cli.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for v in base cur noclaim; do lib $v; timeout 150 python tools/time_encode.py > $OUT/encode_$v.txt 2>&1; done
for v in base cur; do lib $v; timeout 200 python tools/time_e2e.py > $OUT/e2e_$v.txt 2>&1; done
echo done > $OUT/DONE
