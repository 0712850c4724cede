set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
python bench.py --config c4 --steps 20 --warmup 5 > gpurun_out/r2base_c4.json 2> gpurun_out/r2base_c4.err
python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2base_c1.json 2> gpurun_out/r2base_c1.err
for c in c0 c2 c3; do python tools/kbench.py --config $c --iters 30; done > gpurun_out/r2base_kbench.txt 2>&1
( time python bench.py --impl reference --config c4 --steps 3 --warmup 1 ) > gpurun_out/r2base_ref_c4.json 2>&1
