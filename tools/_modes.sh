set -u
for c in c1 c3; do
 for m in 0 1 2; do
  FBF_PLAN_LOG=1 FBF_MODE=$m FBF_LIB=dl/nb.so timeout 300 python tools/kbench.py --config $c --iters 20 --tag mode$m 2>&1 | grep -v "^$" | tail -2
 done
done
