# dev: one GPU call = the driver's tiers (gpu tests, smoke, bench both arms) + the round's profiles.
# usage: bash tools/_r2_round.sh TAG
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
python -m pytest tests -m gpu -x -q --durations=20 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_$TAG.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
bash tools/profile_round.sh $TAG
for c in c0 c1 c2 c3; do
  python bench.py --config $c --steps 50 --warmup 5 --e2e-steps 10 > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "bench $c rc=$?"
done
tail -c 2500 gpurun_out/bench_$TAG.json
