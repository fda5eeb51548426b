#!/bin/bash
# One round of profiles: ncu --set full of each hot kernel, the launch list of the bench, and
# the per-pass R2 metrics of one C5 fwd + bwd.
#   bash tools/profile_round.sh <tag>   (under gpurun; then python tools/ncu_summary.py gpurun_out/ncu <tag>
#                                        and python tools/ncu_passes.py gpurun_out/ncu/passes_<tag>.csv <tag>)
set -x
T=${1:-r2}
D=gpurun_out/ncu
mkdir -p $D
bash tools/ncu_capture.sh k_row_fwd_w c2 $D/${T}_c2_row_fwd --source
bash tools/ncu_capture.sh k_row_bwd_w c2 $D/${T}_c2_row_bwd
bash tools/ncu_capture.sh k_coarse_rows c2 $D/${T}_c2_coarse
bash tools/ncu_capture.sh k_row_fwd_r c5 $D/${T}_c5_row_fwd
bash tools/ncu_capture.sh k_col_fwd c5 $D/${T}_c5_col_fwd
bash tools/ncu_capture.sh k_row_bwd_r c5 $D/${T}_c5_row_bwd
bash tools/ncu_capture.sh k_col_bwd c5 $D/${T}_c5_col_bwd
bash tools/ncu_capture.sh k_plane_fwd c3 $D/${T}_c3_plane_fwd
bash tools/ncu_capture.sh k_plane_bwd c3 $D/${T}_c3_plane_bwd
for c in c5 c4; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_row_fwd|k_col_fwd|k_row_bwd|k_col_bwd" --csv python tools/profile_step.py $c 1 > $D/passes_${T}_$c.csv 2> $D/passes_${T}_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_${T}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-verify > $D/launches_bench.log 2>&1
