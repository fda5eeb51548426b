for v in dyn0_w8 dyn1_w8 dyn1_w14; do echo "== $v"; python tools/ab_lib.py build_ab/$v.so tools/time_2d.py c3 2>&1 | grep -E "fused|bitwise"; done
echo "== HEAD (row direct)"; python tools/time_2d.py c5 c4 2>&1 | grep -E "staged|bitwise"
echo "== HEAD staged rows"; TVP_ROW_DIRECT=0 python tools/time_2d.py c5 c4 2>&1 | grep -E "staged"
