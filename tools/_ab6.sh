for rep in 1 2; do for l in wg wg4896 gw8 cw2; do FBF_LIB=dl/$l.so timeout 200 python tools/kbench.py --config c4 --iters 20 --tag $l; done; done
