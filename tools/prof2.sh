# ncu source-level captures of c1 for two plan variants (dev); usage: bash tools/prof2.sh TAG
mkdir -p gpurun_out
FBF_Q=16 FBF_NGB=2 FBF_NCB=1 ncu --set full --import-source on --clock-control none -k regex:fbf_fused -s 1 -c 1 -o gpurun_out/prof_c1_$1q16 -f python tools/profile_run.py --config c1 > gpurun_out/ncu_q16.log 2>&1
FBF_Q=8 FBF_NGB=2 FBF_NCB=2 ncu --set full --import-source on --clock-control none -k regex:fbf_fused -s 1 -c 1 -o gpurun_out/prof_c1_$1q8 -f python tools/profile_run.py --config c1 > gpurun_out/ncu_q8.log 2>&1
