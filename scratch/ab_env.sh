#!/bin/bash
# same-box A/B of scratch/libs/*.so on the given workloads, with an env setting per run
for w in "$@"; do for v in $(ls scratch/libs | sed 's/.so//'); do echo "$v $w"; python scratch/ab_lib.py scratch/libs/$v.so $w 2>&1 | grep -v stress | head -3; done; done
echo "staged (TVP_FUSED2D=0)"; TVP_FUSED2D=0 python tools/time_kernels.py c3 2>&1 | head -3
