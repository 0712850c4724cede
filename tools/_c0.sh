set -u
for envs in "X=1" "FBF_MODE=0 FBF_Q=16 FBF_NCB=1" "FBF_MODE=0 FBF_Q=16 FBF_NGB=1 FBF_NCB=1" "FBF_MODE=0 FBF_Q=8" "FBF_MODE=1" "FBF_MODE=1 FBF_NCB=1" "FBF_MODE=2"; do
  env $envs FBF_PLAN_LOG=1 timeout 120 python tools/kbench.py --config c0 --iters 40 --tag "$envs" 2>&1 | tail -2
done
