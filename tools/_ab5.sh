set -u
for rep in 1 2 3; do
  FBF_WGQ=8 FBF_LIB=dl/wg.so timeout 300 python tools/kbench.py --config c4 --iters 20 --tag wgq8
  FBF_PLAN_LOG=1 FBF_LIB=dl/wg.so timeout 300 python tools/kbench.py --config c4 --iters 20 --tag wgq16 2>&1 | tail -2
done
python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
