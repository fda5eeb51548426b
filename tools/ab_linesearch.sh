#!/bin/bash
# f3 study: line search every PN iteration (TVP_LS_AFTER=1), sequential
# backtracking vs the parallel four-step search (TVP_LS_PARALLEL=1), against the
# default (projected full Newton steps, line search only after 12 iterations).
#   build here:  bash tools/ab_linesearch.sh build
#   on the GPU:  bash tools/ab_linesearch.sh run     (timings + the full -m gpu suite per variant)
set -e
if [ "$1" == "build" ]; then
  mkdir -p build_ab
  B="python -m paper_2204_03643_b200.build"
  $B --define TVP_LS_AFTER=1 --out build_ab/ls_backtrack.so &
  $B --define TVP_LS_AFTER=1 --define TVP_LS_PARALLEL=1 --out build_ab/ls_parallel.so &
  $B > /dev/null; wait
  cp paper_2204_03643_b200/libtvprox.so build_ab/default.so
  rm -rf paper_2204_03643_b200/build_*
else
  bash tools/ab.sh c2 c5
  cp paper_2204_03643_b200/libtvprox.so /tmp/keep.so
  for v in ls_backtrack ls_parallel; do
    cp build_ab/$v.so paper_2204_03643_b200/libtvprox.so
    echo "$v: $(python -m pytest tests -m gpu -x -q 2>&1 | tail -1)"
  done
  cp /tmp/keep.so paper_2204_03643_b200/libtvprox.so
fi
