set -x
mkdir -p gpurun_out/r3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py > gpurun_out/r3/bench.json 2> gpurun_out/r3/bench.err; echo "bench rc=$?"
bash tools/profile_round.sh ${TAG:-r3b} > gpurun_out/r3/profile.log 2>&1; echo "profile rc=$?"
rm -f gpurun_out/ncu/*.ncu-rep
