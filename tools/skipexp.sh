timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in c1 c3 c4 c2 c0; do timeout 120 python tools/kbench.py --config $c --iters 30 --tag "v22"; done
