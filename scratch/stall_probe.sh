#!/bin/bash
# ncu warp-state stall breakdown of the 1D forward kernel under env settings
for cfg in "TVP_COARSE=1" "TVP_COARSE=0"; do
  env $cfg ncu --section WarpStateStats --section SchedulerStats --section Occupancy --clock-control none -k regex:k_row_fwd_w -s 0 -c 1 --csv --page raw python tools/profile_step.py c2 1 > /tmp/st.csv 2>/dev/null
  echo "== $cfg"
  python3 - <<'PY'
import csv
rows=[r for r in csv.reader(open('/tmp/st.csv')) if len(r)>5]
hdr=rows[0]; val=rows[-1]
for h,v in zip(hdr,val):
    if ('warps_issue_stalled' in h and 'per_issue_active' in h and not h.endswith('not_issued')) or 'issue_active.avg.pct' in h or 'warps_active.avg.pct' in h or 'gpu__time_duration.sum' in h:
        try:
            if float(v) > 0.05: print("  %-90s %s" % (h, v))
        except: pass
PY
done
