# Same-box A/B of variant libraries (under gpurun): a fixed-input bitwise comparison
# (tools/bitcmp.py) and timings (tools/time_kernels.py via tools/ab_lib.py) of every
# build_ab/*.so, then the GPU tests on the in-tree library.
#   AB_WL="c2 c5" [AB_ARGS=...] [AB_NOTEST=1] [AB_REF=<name>] bash tools/ab_run.sh
# Variants: tools/ab_build.sh <rev> <name>, or python -m paper_2204_03643_b200.build
# --define X=Y --out build_ab/<name>.so.
set -x
mkdir -p gpurun_out/ab
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
for v in $(ls build_ab | sed 's/.so//'); do
  python tools/bitcmp.py build_ab/$v.so /tmp/bit_$v.npz > gpurun_out/ab/bit_$v.log 2>&1
done
for w in ${AB_WL:-c2 c5 c3 c4}; do for v in $(ls build_ab | sed 's/.so//'); do
  echo "== $v $w"; python tools/ab_lib.py build_ab/$v.so $w ${AB_ARGS} 2>&1 | grep -v stress | head -4
done; done
for v in $(ls build_ab | sed 's/.so//'); do echo "bitcmp ${AB_REF:-base} vs $v"; python tools/bitcmp_cmp.py /tmp/bit_${AB_REF:-base}.npz /tmp/bit_$v.npz 2>&1 | head -3; done
if [ -z "$AB_NOTEST" ]; then python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x > gpurun_out/ab/t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab/t.log; fi
