# dev: parity + default-plan per-config timing + bench line
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c0 c1 c2 c3 c4; do timeout 120 python tools/kbench.py --config $c --iters 20 --tag default; done
timeout 600 python bench.py > gpurun_out/bench_v17.json 2> gpurun_out/bench_v17.err; tail -1 gpurun_out/bench_v17.json
