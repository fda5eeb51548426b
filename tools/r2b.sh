set -x
timeout 600 python -m pytest tests/test_gpu_parity_2d.py -q -p no:cacheprovider -x -k "fused_plane" > gpurun_out/t2.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/t2.log
timeout 300 python tools/time_2d.py c5 c3 > gpurun_out/t2d.log 2>&1; echo "time rc=$?"; cat gpurun_out/t2d.log | tail -20
TVP_CL_NC14=8 timeout 300 python tools/time_2d.py c5 > gpurun_out/t2d8.log 2>&1; cat gpurun_out/t2d8.log | tail -5
