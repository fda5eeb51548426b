#!/bin/bash
# Capture one kernel with `ncu --set full` and write compact summaries next to it.
#   tools/ncu_capture.sh <kernel-regex> <workload> <out-prefix> [--source]
set -e
K=$1; WL=$2; OUT=$3; SRC=""
if [ "$4" == "--source" ]; then SRC="--import-source on"; fi
ncu --set full --clock-control none $SRC -k regex:$K -s 0 -c 1 -o $OUT python tools/profile_step.py $WL 1 > $OUT.log 2>&1 || true
ncu -i $OUT.ncu-rep --page details --csv > $OUT.details.csv 2>/dev/null || true
ncu -i $OUT.ncu-rep --page raw --csv > $OUT.raw.csv 2>/dev/null || true
if [ -n "$SRC" ]; then ncu -i $OUT.ncu-rep --page source --csv > $OUT.source.csv 2>/dev/null || true; fi
if [ "$(stat -c %s $OUT.ncu-rep 2>/dev/null || echo 0)" -gt 1000000 ]; then rm -f $OUT.ncu-rep; fi
