for v in "16 2 2 1" "8 2 2 2" "16 0 2 2"; do set -- $v
  FBF_Q=$1 FBF_MODE=$2 FBF_NGB=$3 FBF_NCB=$4 timeout 120 python tools/kbench.py --config c1 --iters 30 --tag "Q$1 M$2 $3$4"
done
