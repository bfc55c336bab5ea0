#!/bin/bash
# session 5 re-entry: full GPU suite, smoke and the default bench on the restored tree
set -u
OUT=gpurun_out/r2s5a
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo rc=$? >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo rc=$? >> $OUT/bench.err
timeout 150 python tools/time_encode.py > $OUT/encode.txt 2>&1
echo done > $OUT/DONE
