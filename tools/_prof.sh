# usage: bash tools/_prof.sh LIB CONFIG TAG  (one ncu --set full capture of the fused kernel)
FBF_LIB=$1 python tools/profile_run.py --config $2 > /dev/null 2>&1 && \
FBF_LIB=$1 ncu --set full --import-source on --clock-control none -k regex:fbf_fused -s 2 -c 1 -o gpurun_out/prof_$3 -f \
  python tools/profile_run.py --config $2 > gpurun_out/ncu_$3.log 2>&1; echo ncu_rc=$?
