python tools/time_2d.py c5 c4 2>&1 | grep -E "staged|bitwise"
TVP_ROW_DIRECT=1 timeout 600 python -m pytest tests/test_gpu_parity_2d.py -q -p no:cacheprovider -x 2>&1 | tail -2
echo "== base"; python tools/ab_lib.py build_ab/base.so tools/time_2d.py c5 c4 2>&1 | grep staged
