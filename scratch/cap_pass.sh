#!/bin/bash
# capture one launch of a 2D pass kernel (full set + source) : cap_pass.sh <regex> <skip> <wl> <out>
ncu --set full --import-source on --clock-control none -k regex:$1 -s $2 -c 1 -o $4 python tools/profile_step.py $3 1 > $4.log 2>&1
ncu -i $4.ncu-rep --page raw --csv > $4.raw.csv 2>/dev/null
ncu -i $4.ncu-rep --page source --csv > $4.source.csv 2>/dev/null
rm -f $4.ncu-rep
