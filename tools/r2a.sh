set -x
nvidia-smi -L
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf -x > gpurun_out/t1.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/t1.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke1.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke1.log
timeout 600 python bench.py > gpurun_out/bench1.log 2>gpurun_out/bench1.err; echo "bench rc=$?"; tail -3 gpurun_out/bench1.log; tail -20 gpurun_out/bench1.err
