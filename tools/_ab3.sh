set -u
for c in c0 c1 c2 c4 c3; do
  for rep in 1 2; do
    FBF_LIB=dl/nb2.so timeout 300 python tools/kbench.py --config $c --iters 20 --tag nb2
    FBF_LIB=dl/pdl.so timeout 300 python tools/kbench.py --config $c --iters 20 --tag pdl
    FBF_PDL=0 FBF_LIB=dl/pdl.so timeout 300 python tools/kbench.py --config $c --iters 20 --tag pdl_off
  done
done
python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_host.py -x -q 2>&1 | tail -3
