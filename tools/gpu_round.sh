#!/bin/bash
# One GPU-box pass: parity suite, smoke, bench line, ncu launch list and one
# `ncu --set full` capture of the headline SpMM kernel. Outputs go to
# gpurun_out/ (scratch); copy the summaries worth keeping into profiles/.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag]'
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/smi.txt" 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file "$OUT/launches.csv" python bench.py --quick --steps 3 --warmup 3 > "$OUT/ncu_launch_bench.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_f16_kernel -s 2 -c 1 \
    -o "$OUT/spmm_full" -f python bench.py --quick --steps 3 --warmup 3 > "$OUT/ncu_full.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sddmm_kernel -s 2 -c 1 \
    -o "$OUT/sddmm_full" -f python bench.py --quick --steps 3 --warmup 3 > "$OUT/ncu_full_sddmm.log" 2>&1
echo done > "$OUT/DONE"
