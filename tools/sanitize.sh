#!/bin/bash
# compute-sanitizer memcheck/racecheck over the small GPU tests (run on the GPU box):
#   gpurun --timeout 6000 -- bash tools/sanitize.sh
OUT=gpurun_out/${1:-sanitize}; mkdir -p $OUT
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "known or acceptance6 or baseline16_errors or srbcrs_padding or static_mask or decode or taxonomy" > $OUT/memcheck_parity.log 2>&1; echo "rc=$?" >> $OUT/memcheck_parity.log
timeout 1800 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_layers.py tests/test_gpu_scale.py -m gpu -q -x -k "not config3 and not config5 and not midsize" > $OUT/memcheck_layers.log 2>&1; echo "rc=$?" >> $OUT/memcheck_layers.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "known_answer" > $OUT/racecheck.log 2>&1; echo "rc=$?" >> $OUT/racecheck.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_layers.py -m gpu -q -x -k "attend or aggregate" > $OUT/racecheck_layers.log 2>&1; echo "rc=$?" >> $OUT/racecheck_layers.log
# round 2: the pipelined host-buffer path (sync-free chunk encode, side streams) and its late-chunk errors
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_scale.py -m gpu -q -x -k "pipelined or midsize" > $OUT/memcheck_pipeline.log 2>&1; echo "rc=$?" >> $OUT/memcheck_pipeline.log
# round 2: the small-list burst kernels (shared-memory part reduction, PDL launches)
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "known_answer or config1 or acceptance2" > $OUT/racecheck_burst.log 2>&1; echo "rc=$?" >> $OUT/racecheck_burst.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "known_answer or config1" > $OUT/synccheck_burst.log 2>&1; echo "rc=$?" >> $OUT/synccheck_burst.log
