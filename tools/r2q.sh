echo "== HEAD w8"; python tools/time_2d.py c5 2>&1 | grep staged
for v in f4m4 f4m3 f2m8; do echo "== $v"; python tools/ab_lib.py build_ab/$v.so tools/time_2d.py c5 2>&1 | grep -E "staged"; done
