echo "== m2 (HEAD)"; python tools/time_2d.py c3 2>&1 | grep fused; for v in m3 m4; do echo "== $v"; python tools/ab_lib.py build_ab/$v.so tools/time_2d.py c3 2>&1 | grep -E "fused"; done
