#!/bin/bash
# session 5: AGNN attention issue without the zero-select on loaded data (cur) vs before (base): layer tests,
# tools/time_attend.py interleaved; the default bench with the new TF32 sub-object
set -u
OUT=gpurun_out/r2s5f
mkdir -p $OUT
lib() { if [ "$1" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$1/libtcsparse_b200.so; fi; }
lib cur; timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_fullsize.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2; do for v in base cur; do lib $v; timeout 200 python tools/time_attend.py > $OUT/attend_${v}_$r.txt 2>&1; done; done
lib cur; timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo rc=$? >> $OUT/bench.err
echo done > $OUT/DONE
