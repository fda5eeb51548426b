D=gpurun_out/ncu; mkdir -p $D
for c in c5 c4; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_row_fwd|k_col_fwd|k_row_bwd|k_col_bwd" --csv python tools/profile_step.py $c 1 > $D/passes_r2m_$c.csv 2> $D/passes_r2m_$c.err
done
ls -la $D | tail -4
