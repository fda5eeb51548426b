timeout 900 python -m pytest tests/test_gpu_parity_2d.py tests/test_gpu_parity_1d.py tests/test_gpu_determinism.py -q -p no:cacheprovider -x 2>&1 | tail -3
echo "== stream"; python tools/time_2d.py c5 2>&1 | grep -E "staged|bitwise"
echo "== no stream"; TVP_ROW_STREAM=0 python tools/time_2d.py c5 2>&1 | grep -E "staged"
echo "== C3 staged stream vs not (fused off)"; python tools/time_2d.py c3 2>&1 | grep staged; TVP_ROW_STREAM=0 python tools/time_2d.py c3 2>&1 | grep staged
