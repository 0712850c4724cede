# Round profiling pass (1 GPU): bench line, launch list of the same command, and
# full ncu captures of the fused kernel for c1 / c4 / c2. Usage: bash tools/profile_round.sh TAG
set -u
TAG=${1:-rNN}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err && tail -1 gpurun_out/bench_$TAG.json
python bench.py --steps 20 --warmup 3 --e2e-steps 5 --no-cpu-baseline > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:fbf_fused -c 60 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 20 --warmup 3 --e2e-steps 5 --no-cpu-baseline > gpurun_out/ncu_launches_$TAG.log 2>&1
for c in c1 c4 c2; do
  python tools/profile_run.py --config $c > gpurun_out/plain_$c.log 2>&1 &&
  ncu --set full --import-source on --clock-control none -k regex:fbf_fused -s 1 -c 1 -o gpurun_out/prof_${c}_$TAG -f \
      python tools/profile_run.py --config $c > gpurun_out/ncu_${c}_$TAG.log 2>&1
done
ls gpurun_out/*$TAG*
