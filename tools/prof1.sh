# ncu source-level capture of c1 with a given plan (dev); usage: Q MODE NGB NCB TAG
mkdir -p gpurun_out
FBF_Q=$1 FBF_MODE=$2 FBF_NGB=$3 FBF_NCB=$4 ncu --set full --import-source on --clock-control none -k regex:fbf_fused -s 1 -c 1 -o gpurun_out/prof_c1_$5 -f python tools/profile_run.py --config c1 > gpurun_out/ncu_$5.log 2>&1
