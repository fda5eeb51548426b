timeout 900 python -m pytest tests/test_gpu_parity_1d.py -q -p no:cacheprovider -x -k "cluster or limit or long" 2>&1 | tail -4
python tools/time_kernels.py long 8192 16384 32768 65536 131072 2>&1 | tail -6
