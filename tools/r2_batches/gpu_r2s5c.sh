#!/bin/bash
# session 5: TF32 value conversion moved from issue to compute (cur) vs HEAD (base): TF32 parity tests,
# C3 TF32 N=64/128/256 timing (interleaved, twice); small configs incl. SDDMM burst warps-per-item caps
set -u
OUT=gpurun_out/r2s5c
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_scale.py -m gpu -x -q -k "tf32 or TF32 or f32" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2; do for v in base cur; do lib $v; timeout 200 python tools/time_tf32.py > $OUT/tf32_${v}_$r.txt 2>&1; done; done
for v in base cur sub4 sub6 g4s3 g1; do lib $v; timeout 200 python tools/time_small.py 3 > $OUT/small_$v.txt 2>&1; done
echo done > $OUT/DONE
