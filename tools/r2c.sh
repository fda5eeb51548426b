timeout 600 python -m pytest tests/test_gpu_parity_2d.py -q -p no:cacheprovider -x -k "fused_plane" 2>&1 | tail -3
for v in cl1 cl0; do echo "== $v"; TVP_CL_VERBOSE=1 python tools/ab_lib.py build_ab/$v.so tools/time_2d.py c5 2>&1 | grep -v "^$" | tail -4; done
echo "== NC14=8"; TVP_CL_NC14=8 TVP_CL_VERBOSE=1 python tools/time_2d.py c5 2>&1 | tail -4
