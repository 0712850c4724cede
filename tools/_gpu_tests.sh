# dev: the driver's GPU tiers in one call (tests, smoke, bench c4 + reference arm)
python -m pytest tests -m gpu -x -q --durations=15 -s > gpurun_out/pytest_gpu_r2.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu_r2.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_r2a.json
