D=gpurun_out/ncu; mkdir -p $D
ncu --set full --clock-control none --import-source on -k regex:k_row_fwd_w -s 1 -c 1 -o $D/r2f_c2_fwd python tools/profile_step.py c2 2 > $D/r2f.log 2>&1
ncu -i $D/r2f_c2_fwd.ncu-rep --page source --csv --print-source sass > $D/r2f_c2_fwd.sass.csv 2>/dev/null
ncu -i $D/r2f_c2_fwd.ncu-rep --page source --csv --print-source cuda > $D/r2f_c2_fwd.cuda.csv 2>/dev/null
ncu -i $D/r2f_c2_fwd.ncu-rep --page raw --csv > $D/r2f_c2_fwd.raw.csv 2>/dev/null
rm -f $D/r2f_c2_fwd.ncu-rep
ls -la $D
