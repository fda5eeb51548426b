python tools/sanitize.py && echo plain-ok
for t in memcheck synccheck; do echo "== $t"; timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/san_$t.txt 2>&1; echo "rc=$?"; tail -3 gpurun_out/san_$t.txt; done
for t in racecheck initcheck; do echo "== $t"; timeout 1800 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py quick > gpurun_out/san_$t.txt 2>&1; echo "rc=$?"; tail -3 gpurun_out/san_$t.txt; done
