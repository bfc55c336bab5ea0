#!/bin/bash
# A/B timing of library builds on one GPU box: for each NAME, variants/NAME
# (tools/build_variant.sh) or "cur" (the in-tree build), run the small-config,
# per-op and layer timing aids.  Outputs: gpurun_out/ab_<tag>/<NAME>.*
#   gpurun -- 'bash tools/ab.sh TAG NAME1 NAME2 ...'
set -u
TAG=$1; shift
OUT=gpurun_out/ab_$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$OUT/smi.txt" 2>&1
for v in "$@"; do
  if [ "$v" = cur ]; then unset TCS_LIB_PATH; else export TCS_LIB_PATH=$PWD/variants/$v/libtcsparse_b200.so; fi
  timeout 300 python tools/time_small.py 3 > "$OUT/$v.small" 2>&1
  timeout 600 python tools/time_ops.py ${AB_OPS:-c3 c4 c5} > "$OUT/$v.ops" 2>&1
  [ -n "${AB_LAYERS:-1}" ] && timeout 600 python tools/bench_layers.py > "$OUT/$v.layers" 2>&1
done
echo done > "$OUT/DONE"
