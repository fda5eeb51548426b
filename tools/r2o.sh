echo "== w8 (HEAD)"; python tools/time_2d.py c4 2>&1 | grep staged
for v in c16w4 c16w2; do echo "== $v"; python tools/ab_lib.py build_ab/$v.so tools/time_2d.py c4 2>&1 | grep -E "staged"; done
python tools/pairwaste.py
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-verify > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_r2z.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-verify > /dev/null 2>&1
