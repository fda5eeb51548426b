echo "== minb6 (HEAD)"; python tools/time_2d.py c5 c4 2>&1 | grep -E "staged"
for v in cbm4 cbm8; do echo "== $v"; python tools/ab_lib.py build_ab/$v.so tools/time_2d.py c5 c4 2>&1 | grep -E "staged"; done
