#!/bin/bash
# ncu captures of one call per operator/config (tools/profile_ops.py under
# --profile-from-start off).  Each report is exported on the box to its raw
# metrics CSV and a text summary (tools/ncu_summary.py); the .ncu-rep itself
# is kept only if KEEP_REP=1 (reports are large; gpurun_out/ must stay under
# 64 MiB).  Then tools/traffic_from_ncu.py can be run on the CSVs.
#   gpurun -- 'bash tools/gpu_profiles.sh TAG [cfg:op:prec:width ...]'
set -u
TAG=${1:-prof}; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
SPECS=${@:-"c1:spmm:fp16:128 c1:sddmm:fp16:32 c3:spmm:fp16:128 c3:spmm:tf32:128 c3:sddmm:fp16:32 c4:spmm:fp16:128 c5:spmm:fp16:32 c5:sddmm_static:fp16:32"}
for spec in $SPECS; do
  IFS=: read cfg op prec w <<< "$spec"
  name=${cfg}_${op}_${prec}_${w}
  rep=/tmp/ncu_$name
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -o "$rep" -f python tools/profile_ops.py $cfg $op $prec $w > "$OUT/$name.log" 2>&1
  echo "$name rc=$?" >> "$OUT/status.txt"
  ncu -i "$rep.ncu-rep" --page raw --csv > "$OUT/$name.raw.csv" 2>> "$OUT/$name.log"
  python tools/ncu_summary.py "$OUT/$name.raw.csv" > "$OUT/$name.summary.txt" 2>> "$OUT/$name.log"
  if [ "${KEEP_REP:-0}" = 1 ]; then cp "$rep.ncu-rep" "$OUT/"; fi
  rm -f "$rep.ncu-rep"
done
