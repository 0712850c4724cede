for lib in c2 g3 g3c2; do FBF_LIB=devlib/$lib.so timeout 120 python tools/kbench.py --config c1 --tag "$lib"; done
timeout 120 python tools/kbench.py --config c1 --tag "base"
