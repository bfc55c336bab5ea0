#!/bin/bash
# session 5: f32-stored FP16 values converted at the MMA in the 128-feature kernels (cur, TCS_VF32_DEFER=1) vs at the
# load (nodefer): parity on cur (every golden case with f32 value storage), C3 timing interleaved
set -u
OUT=gpurun_out/r2s5i
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_dropin.py tests/test_gpu_fullsize.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2; do for v in nodefer cur; do lib $v; timeout 300 python tools/time_vf32.py > $OUT/vf32_${v}_$r.txt 2>&1; done; done
echo done > $OUT/DONE
