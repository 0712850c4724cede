for v in "16 0" "8 0" "8 1"; do set -- $v
  for pc in 1 2 4 8 16; do echo -n "Q$1 M$2 pieces "; FBF_Q=$1 FBF_MODE=$2 FBF_PIECES=$pc timeout 120 python tools/e2e_probe.py; done
done
