set -u
for c in c4; do
  for rep in 1 2 3; do
    FBF_HALF_SPLIT=0 FBF_LIB=dl/wg.so timeout 300 python tools/kbench.py --config $c --iters 20 --tag nosplit
    FBF_LIB=dl/wg.so timeout 300 python tools/kbench.py --config $c --iters 20 --tag wgsplit
  done
done
python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
