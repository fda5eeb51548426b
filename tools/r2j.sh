timeout 900 python -m pytest tests/test_gpu_parity_2d.py tests/test_gpu_determinism.py tests/test_gpu_layer.py -q -p no:cacheprovider -x 2>&1 | tail -2
python tools/time_2d.py c5 c4 2>&1 | grep -E "staged|bitwise"
