timeout 900 python -m pytest tests/test_gpu_parity_2d.py -q -p no:cacheprovider -x 2>&1 | tail -2
echo "== stream"; python tools/time_2d.py c3 2>&1 | grep -E "fused|bitwise"
echo "== lockstep"; TVP_PLANE_STREAM=0 python tools/time_2d.py c3 2>&1 | grep -E "fused"
