# dev: kbench A/B of env settings over configs. usage: bash tools/_ab.sh "ENV1" "ENV2" -- c4 c1 ...
set -u
A=$1; B=$2; shift 3
for c in "$@"; do
  for rep in 1 2; do
    env $A timeout 300 python tools/kbench.py --config $c --iters 20 --tag "A:$A" 
    env $B timeout 300 python tools/kbench.py --config $c --iters 20 --tag "B:$B"
  done
done
