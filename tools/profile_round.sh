#!/bin/bash
# One round of profiles: ncu --set full of each hot kernel + the launch list of the bench.
#   bash tools/profile_round.sh <tag>   (under gpurun; then python tools/ncu_summary.py gpurun_out/ncu <tag>)
set -x
T=${1:-r1f}
D=gpurun_out/ncu
mkdir -p $D
bash tools/ncu_capture.sh k_row_fwd_w c2 $D/${T}_c2_row_fwd --source
bash tools/ncu_capture.sh k_row_bwd_w c2 $D/${T}_c2_row_bwd
bash tools/ncu_capture.sh k_coarse_rows c2 $D/${T}_c2_coarse
bash tools/ncu_capture.sh k_row_fwd c5 $D/${T}_c5_row_fwd
bash tools/ncu_capture.sh k_col_fwd c5 $D/${T}_c5_col_fwd
bash tools/ncu_capture.sh k_row_bwd c5 $D/${T}_c5_row_bwd
bash tools/ncu_capture.sh k_col_bwd c5 $D/${T}_c5_col_bwd
bash tools/ncu_capture.sh k_plane_fwd c3 $D/${T}_c3_plane_fwd
bash tools/ncu_capture.sh k_plane_bwd c3 $D/${T}_c3_plane_bwd
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_${T}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $D/launches_bench.log 2>&1
