timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 300 python tools/time_2d.py c5 c3 2>&1 | tail -6
